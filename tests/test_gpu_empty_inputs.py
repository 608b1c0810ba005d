"""Empty and degenerate inputs through the public entry points, against the
oracle's behaviour for the same inputs (the reference's edge semantics):

  * nn_query (_kernels/_numpy.py:65-138): empty query, empty reference
    (inf / -1), a single reference point;
  * inverse_project (backend.py:78-101): all-invalid frames give no points;
    one valid pixel gives exactly that point;
  * match_batched (tracking.py:143-170 per pair): pairs with an empty side
    next to a regular pair in one launch;
  * update_similarity scoring (loops.py:184-243): databases smaller than the
    exclusion window admit nothing.
"""

import numpy as np
import pytest
import torch

from oracle import kernels as okern
from oracle import ref_numpy as ref

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs CUDA")


def test_nn_query_empty_and_single():
    from paper_2510_02080_b200 import kernels

    rng = np.random.default_rng(0)
    q = rng.random((50, 3))
    r = rng.random((40, 3))
    for qq, rr in ((np.zeros((0, 3)), r), (q, np.zeros((0, 3))), (q, r[:1]), (q[:1], r)):
        d, i = kernels.nn_query(qq, rr, 0.05)
        de, ie = okern.nn_query(qq, rr, 0.05)
        assert d.shape == de.shape and i.shape == ie.shape
        np.testing.assert_array_equal(i, ie)
        np.testing.assert_array_equal(d, de)


def test_inverse_project_all_invalid_and_single_pixel():
    from paper_2510_02080_b200 import backend

    F, H, W = 2, 12, 20
    K4 = np.array([30.0, 30.0, 9.5, 5.5])
    poses = np.tile(np.array([1.0, 1.0, 0, 0, 0, 0, 0, 0]), (F, 1))
    poses[1, 5:] = (0.1, -0.2, 0.3)
    depth = np.zeros((F, H, W), np.float32)
    conf = np.zeros_like(depth)
    pts, cf, fid, pix = backend.inverse_project_device(torch.as_tensor(depth, device="cuda"),
                                                       torch.as_tensor(conf, device="cuda"), K4, poses, [3, 7])
    assert pts.shape == (0, 3) and cf.shape == (0,) and fid.shape == (0,) and pix.shape == (0, 2)
    depth[1, 4, 17] = 2.5
    conf[1, 4, 17] = 0.75
    got = [x.cpu().numpy() for x in backend.inverse_project_device(
        torch.as_tensor(depth, device="cuda"), torch.as_tensor(conf, device="cuda"), K4, poses, [3, 7])]
    exp = ref.inverse_project(depth, conf, [3, 7], poses[:, 1:5], poses[:, 5:], K4)
    for g, e in zip(got, exp):
        np.testing.assert_array_equal(g, e)


def test_match_batched_pairs_with_empty_sides():
    from paper_2510_02080_b200 import tracking

    rng = np.random.default_rng(1)

    def unit(n, d=64):
        x = rng.normal(size=(n, d))
        return x / np.linalg.norm(x, axis=1, keepdims=True)

    A, B = unit(200), unit(180)
    pairs = [(A, np.zeros((0, 64))), (np.zeros((0, 64)), B), (A, B), (A[:1], B), (A, B[:1])]
    got = tracking.match_batched(pairs, 0.8)
    assert len(got) == len(pairs)
    for (a, b), g in zip(pairs, got):
        exp = ref.match_descriptors_vec(a, b, 0.8) if len(a) and len(b) else np.zeros((0, 2), np.int64)
        np.testing.assert_array_equal(np.asarray(g).reshape(-1, 2), np.asarray(exp).reshape(-1, 2))
    assert tracking.match_descriptors(np.zeros((0, 64)), B, 0.8) == []


@pytest.mark.parametrize("K", [1, 5, 15, 16])
def test_retrieval_small_databases(K):
    from paper_2510_02080_b200 import loops

    rng = np.random.default_rng(K)
    pooled = rng.normal(size=(K, 64))
    pooled /= np.linalg.norm(pooled, axis=1, keepdims=True)
    pooled[1:] = pooled[:1] + 0.01 * pooled[1:]  # near-duplicates: every score above both thresholds
    pooled /= np.linalg.norm(pooled, axis=1, keepdims=True)
    st = ref.SimilarityState()
    kfs = np.arange(K) * 5
    exp = ref.update_similarity(st, kfs, pooled, 5, 15, 0.93, 0.96)
    cp, cs, qp, qs, ep, es = loops.retrieval_device(torch.as_tensor(pooled, device="cuda"), 5, 15, 0.93, 0.96)
    adm = loops.admit(loops.SimilarityMatrix(), kfs, qp, qs)
    assert [p for p, _ in adm] == [p for p, _ in exp]
    if K <= 15:
        assert exp == []  # every pair inside the exclusion window
