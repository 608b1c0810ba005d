"""Drop-in wrappers called directly with the reference's own objects (the
unmodified reference from baseline/_ref), result against the reference
function on the same inputs:

  * registration.normalize_confidences / weighted_umeyama
    (registration.py:28-35,105-112) incl. their error precedence;
  * tracking.match_to_map (tracking.py:173-194) on a reference
    LocalSparseMap / FrameObservation;
  * mapping.b200_mapping_class(Mapping) (mapping.py:114-211,332-338):
    build_submap -> register_submap over three flushes and fused_cloud,
    against the reference Mapping on the same SyntheticBackend.

The reference's whole suites also run through binding.install()
(tests/test_gpu_reference_suite.py); these tests pin the wrappers one by one.
"""

import os
import sys

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")
if not os.path.isdir(os.path.join(REF, "submap_slam")):
    pytest.skip("reference not installed in baseline/_ref", allow_module_level=True)
if REF not in sys.path:
    sys.path.append(REF)

from submap_slam import registration as rreg  # noqa: E402
from submap_slam import tracking as rtrk  # noqa: E402

from paper_2510_02080_b200 import registration as breg  # noqa: E402
from paper_2510_02080_b200 import tracking as btrk  # noqa: E402


@pytest.fixture(autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs CUDA")


def _raises_same(fn_ref, fn_ours, *args):
    with pytest.raises(Exception) as e_ref:
        fn_ref(*args)
    with pytest.raises(Exception) as e_ours:
        fn_ours(*args)
    assert type(e_ours.value).__name__ == type(e_ref.value).__name__


def test_normalize_confidences_matches_reference():
    rng = np.random.default_rng(0)
    for n in (1, 3, 1000):
        c = rng.random(n)
        np.testing.assert_array_equal(breg.normalize_confidences(c), rreg.normalize_confidences(c))
    z = [0.0, 2.0, 0.0]
    np.testing.assert_array_equal(breg.normalize_confidences(z), rreg.normalize_confidences(z))
    for bad in ([], [0.0, 0.0], [-1.0, 2.0], [-1.0, 0.0]):
        _raises_same(rreg.normalize_confidences, breg.normalize_confidences, bad)


def _sim3_close(a, b, rtol=1e-5):
    assert abs(a.scale - b.scale) <= rtol * abs(b.scale)
    qa, qb = np.asarray(a.rotation.q, float), np.asarray(b.rotation.q, float)
    if np.dot(qa, qb) < 0:
        qa = -qa
    np.testing.assert_allclose(qa, qb, atol=rtol)
    np.testing.assert_allclose(np.asarray(a.translation), np.asarray(b.translation),
                               atol=rtol * max(1.0, float(np.abs(b.translation).max())))


def test_weighted_umeyama_matches_reference():
    rng = np.random.default_rng(1)
    for n in (3, 10, 500):
        p = rng.normal(size=(n, 3))
        ang = rng.normal(size=3)
        th = np.linalg.norm(ang)
        k = ang / th
        K = np.array([[0, -k[2], k[1]], [k[2], 0, -k[0]], [-k[1], k[0], 0]])
        R = np.eye(3) + np.sin(th) * K + (1 - np.cos(th)) * K @ K
        q = 1.7 * p @ R.T + rng.normal(size=3) + 1e-3 * rng.normal(size=(n, 3))
        w = rng.random(n) + 0.05
        corrs = [rreg.Correspondence3D3D(p[i], q[i], float(w[i])) for i in range(n)]
        t_ref, rms_ref = rreg.weighted_umeyama(corrs)
        t_ours, rms_ours = breg.weighted_umeyama(corrs)
        _sim3_close(t_ours, t_ref)
        assert abs(rms_ours - rms_ref) <= 1e-6 * max(rms_ref, 1e-9)
    p = rng.normal(size=(2, 3))
    _raises_same(rreg.weighted_umeyama, breg.weighted_umeyama,
                 [rreg.Correspondence3D3D(p[i], p[i], 1.0) for i in range(2)])
    p = rng.normal(size=(5, 3))
    _raises_same(rreg.weighted_umeyama, breg.weighted_umeyama,
                 [rreg.Correspondence3D3D(p[i], p[i], 0.0) for i in range(5)])


def _unit(rng, n, d):
    x = rng.normal(size=(n, d))
    return x / np.linalg.norm(x, axis=1, keepdims=True)


def test_match_to_map_matches_reference():
    rng = np.random.default_rng(2)
    for n_map, n_obs, d in ((300, 250, 64), (1024, 1024, 256), (1, 5, 64)):
        desc = _unit(rng, n_map, d)
        sm = rtrk.LocalSparseMap()
        sm.insert_batch([rtrk.SparseMapPoint(id=sm.allocate_id(), position=rng.normal(size=3), descriptor=desc[i],
                                             confidence=0.5, source_keyframe=0) for i in range(n_map)])
        pick = rng.choice(n_map, size=min(n_obs, n_map), replace=False)
        od = desc[pick] + 0.05 * rng.normal(size=(len(pick), d))
        od = np.concatenate([od, _unit(rng, n_obs - len(pick), d)])
        od /= np.linalg.norm(od, axis=1, keepdims=True)
        obs = rtrk.FrameObservation(frame_id=7, keypoints=rng.random((n_obs, 2)) * 500, descriptors=od)
        cfg = rtrk.TrackingConfig()
        c_ref, i_ref, p_ref = rtrk.match_to_map(obs, sm, cfg)
        c_ours, i_ours, p_ours = btrk.match_to_map(obs, sm, cfg)
        np.testing.assert_array_equal(i_ours, i_ref)
        np.testing.assert_array_equal(p_ours, p_ref)
        assert len(c_ours) == len(c_ref) > 0
        for a, b in zip(c_ours, c_ref):
            np.testing.assert_array_equal(a.pixel, b.pixel)
            np.testing.assert_array_equal(a.point, b.point)
            assert a.point_id == b.point_id
    empty = rtrk.LocalSparseMap()
    obs = rtrk.FrameObservation(frame_id=0, keypoints=np.zeros((3, 2)), descriptors=_unit(rng, 3, 64))
    c, i, p = btrk.match_to_map(obs, empty, rtrk.TrackingConfig())
    assert c == [] and len(i) == 0 and len(p) == 0


def test_b200_mapping_class_matches_reference_mapping():
    from submap_slam.backend import SyntheticBackend, SyntheticBackendConfig
    from submap_slam.loops import FlushBatch
    from submap_slam.mapping import Mapping
    from submap_slam.scenesim import TrajectorySpec, WorldConfig, generate_trajectory, generate_world

    from paper_2510_02080_b200.mapping import b200_mapping_class

    def backend():
        world = generate_world(WorldConfig(room_size=(8.0, 8.0, 4.0), landmark_count=300), 0)
        traj = generate_trajectory(TrajectorySpec(kind="circle", frame_count=16, radius=2.0, step_bound=1.0), world)
        return SyntheticBackend(world, traj, SyntheticBackendConfig(), seed=100)

    batches = [FlushBatch(new_ids=(0, 1, 2, 3, 4), old_ids=()), FlushBatch(new_ids=(5, 6, 7, 8), old_ids=(4,)),
               FlushBatch(new_ids=(9, 10, 11, 12), old_ids=(8,))]
    ref_mp = Mapping(backend())
    ours = b200_mapping_class(Mapping)(backend())
    for b in batches:
        s_ref = ref_mp.register_submap(ref_mp.build_submap(b))
        s_ours = ours.register_submap(ours.build_submap(b))
        assert s_ours.edges_added == s_ref.edges_added
    for a, b in zip(ours.submaps.values(), ref_mp.submaps.values()):
        assert a.keyframe_ids == b.keyframe_ids
        _sim3_close(a.global_pose, b.global_pose)
    x_ref, c_ref = ref_mp.fused_cloud()
    x_ours, c_ours = ours.fused_cloud()
    # the device pool holds float32 depth / confidence planes (SURVEY §8(a) a1:
    # inputs cast to fp32), so the concatenated cloud matches to fp32 rounding
    assert x_ours.shape == x_ref.shape
    np.testing.assert_allclose(c_ours, c_ref, rtol=2.0 ** -23, atol=0)
    assert float(np.abs(x_ours - x_ref).max()) < 1e-6
