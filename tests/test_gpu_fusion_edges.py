"""Voxel fusion edge cases against the oracle (oracle/fuse.py, the declared
rule over mapping.py:56-57,332-338 and _kernels/_numpy.py:50-55):

  * a submap whose every pixel is invalid (depth 0): an empty map;
  * points exactly on voxel faces and one float32 ulp either side (depths at
    float32(cell * k) and their neighbours, the principal column / row on
    x = 0 / y = 0), which the kernel's float32 fast path must hand to its
    exact float64 path: keys and counts bit-exact;
  * depth > 0 with confidence 0 (dropped by the rule's conf > 0) mixed with
    an all-invalid frame inside one submap.
"""

import numpy as np
import pytest
import torch

from oracle import fuse as ofuse

pytestmark = pytest.mark.gpu

H, W = 48, 64
K4 = np.array([50.0, 50.0, 32.0, 24.0])  # integer principal point: pixels on x = 0 / y = 0
CELL = 0.02
IDENT = (1.0, np.array([1.0, 0.0, 0.0, 0.0]), np.zeros(3))


@pytest.fixture(autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs CUDA")


def _fuse(depth, conf, poses8):
    from paper_2510_02080_b200 import mapping

    F = depth.shape[0]
    dm = mapping.DenseMapping(H, W, K4)
    ids = list(range(F))
    sm = dm.add_submap(ids, torch.as_tensor(depth, device="cuda"), torch.as_tensor(conf, device="cuda"), list(poses8))
    dm.register_chain([sm])  # the first submap: the fixed root, identity global pose
    out = dm.fused_cloud(voxel=CELL)
    dense = [dict(depth=depth, conf=conf, frame_ids=np.array(ids), pose_q=poses8[:, 1:5], pose_t=poses8[:, 5:],
                  K=K4)]
    return out, ofuse.fuse_submaps(dense, [IDENT], CELL)


def _poses(F, rng):
    p = np.zeros((F, 8))
    p[:, 0] = 1.0
    p[:, 1] = 1.0
    for f in range(1, F):  # small rotations / translations for the later frames
        q = np.array([1.0, *(0.01 * rng.normal(size=3))])
        p[f, 1:5] = q / np.linalg.norm(q)
        p[f, 5:] = 0.05 * rng.normal(size=3)
    return p


def _check(out, o):
    np.testing.assert_array_equal(out["keys"], o["keys"])
    np.testing.assert_array_equal(out["count"], o["count"])
    if len(o["keys"]):
        assert np.max(np.abs(out["centroid"] - o["centroid"])) < 1e-4
        np.testing.assert_allclose(out["wsum"], o["wsum"], rtol=1e-4)
    assert out["stats"]["n_points_in"] == o["n_in"]


def test_all_invalid_submap_is_empty():
    depth = np.zeros((3, H, W), np.float32)
    conf = np.zeros_like(depth)
    out, o = _fuse(depth, conf, _poses(3, np.random.default_rng(0)))
    assert len(o["keys"]) == 0 and len(out["keys"]) == 0
    _check(out, o)


def test_face_aligned_depths_take_the_exact_path():
    rng = np.random.default_rng(1)
    v, u = np.mgrid[0:H, 0:W]
    k = 40 + (u + 3 * v) % 23
    base = (CELL * k).astype(np.float32)  # float32(cell * k): on or next to a z face
    depth = np.stack([base, np.nextafter(base, np.float32(np.inf)), np.nextafter(base, np.float32(0))])
    conf = rng.uniform(0.1, 1.0, size=depth.shape).astype(np.float32)
    poses = np.zeros((3, 8))
    poses[:, 0] = 1.0
    poses[:, 1] = 1.0  # identity: x = (u - 32) z / 50 lands on x faces too
    out, o = _fuse(depth, conf, poses)
    _check(out, o)
    assert out["stats"]["n_slow_path"] > 0  # the float64 face path ran


def test_zero_confidence_and_invalid_frame_mixed():
    rng = np.random.default_rng(2)
    depth = rng.uniform(0.8, 3.0, size=(4, H, W)).astype(np.float32)
    conf = rng.uniform(0.05, 1.0, size=depth.shape).astype(np.float32)
    depth[1] = 0.0
    conf[1] = 0.0                              # frame 1: nothing valid
    conf[2][rng.random((H, W)) < 0.5] = 0.0    # frame 2: depth > 0 but conf 0 -> dropped
    depth[3][rng.random((H, W)) < 0.3] = 0.0   # frame 3: holes
    conf[3][depth[3] == 0] = 0.0
    out, o = _fuse(depth, conf, _poses(4, rng))
    assert o["n_in"] == int(((depth > 0) & (conf > 0)).sum())
    _check(out, o)
