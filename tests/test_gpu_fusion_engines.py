"""The binned super-block fusion engine (csrc/vbin.cu, EC3R_FUSE_ENGINE=binned)
against the oracle's declared fusion rule (oracle/fuse.py, keys
_kernels/_numpy.py:50-55 of the mapping.py:56-57 transform) and against the
default block-hash engine; its integer accumulation makes it bit-for-bit
deterministic and independent of the insertion split."""

import numpy as np
import pytest
import torch

from oracle import fuse as ofuse
from tests.conftest import mapping_submaps

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs CUDA")


@pytest.fixture
def binned(monkeypatch):
    monkeypatch.setenv("EC3R_FUSE_ENGINE", "binned")


def _registered(g):
    from paper_2510_02080_b200 import mapping
    sms_g, _ = mapping_submaps(g)
    K4 = sms_g[0]["K"]
    H, W = sms_g[0]["depth"].shape[1:]
    dm = mapping.DenseMapping(H, W, K4)
    sms = []
    for s in sms_g:
        poses8 = np.concatenate([np.ones((len(s["frame_ids"]), 1)), s["pose_q"], s["pose_t"]], axis=1)
        sms.append(dm.add_submap(s["frame_ids"], s["depth"], s["conf"], list(poses8)))
    dm.register_chain(sms)
    return dm, sms, sms_g


def _globs(sms):
    return [(sm.global_pose.scale, np.asarray(sm.global_pose.rotation.q), np.asarray(sm.global_pose.translation))
            for sm in sms]


def test_binned_fusion_vs_oracle(golden, binned):
    g = golden("mapping")
    dm, sms, sms_g = _registered(g)
    for cell in (0.02, 0.05, 0.013):
        dm._vmap = None
        out = dm.fused_cloud(voxel=cell)
        o = ofuse.fuse_submaps(sms_g, _globs(sms), cell)
        np.testing.assert_array_equal(out["keys"], o["keys"])
        np.testing.assert_array_equal(out["count"], o["count"])
        np.testing.assert_allclose(out["wsum"], o["wsum"], rtol=1e-5)
        assert np.max(np.abs(out["centroid"] - o["centroid"])) < 1e-4
        assert out["stats"]["n_points_in"] == o["n_in"]


def test_binned_deterministic_and_split_invariant(golden, binned):
    """Integer fixed-point sums: two fills, and one-shot vs slot-by-slot
    insertion, give bit-identical keys, centroids, wsum and counts."""
    from paper_2510_02080_b200 import mapping
    g = golden("mapping")
    dm, sms, _ = _registered(g)
    slots = dm.all_slots()
    a = mapping.VoxelMap(0.02, 1 << 19)
    a.insert_frames(dm.pool, slots)
    r1 = [x.cpu().numpy() for x in a.extract()]
    a.clear()
    a.insert_frames(dm.pool, slots)
    r2 = [x.cpu().numpy() for x in a.extract()]
    b = mapping.VoxelMap(0.02, 1 << 19)
    for s in range(slots.numel()):
        b.insert_frames(dm.pool, slots[s:s + 1])
    r3 = [x.cpu().numpy() for x in b.extract()]
    for x, y, z in zip(r1, r2, r3):
        np.testing.assert_array_equal(x, y)
        np.testing.assert_array_equal(x, z)


def test_binned_equals_block_hash_engine(golden, monkeypatch):
    from paper_2510_02080_b200 import mapping
    g = golden("mapping")
    dm, sms, _ = _registered(g)
    slots = dm.all_slots()
    monkeypatch.setenv("EC3R_FUSE_ENGINE", "binned")
    a = mapping.VoxelMap(0.02, 1 << 19)
    monkeypatch.delenv("EC3R_FUSE_ENGINE")
    b = mapping.VoxelMap(0.02, 1 << 19)
    a.insert_frames(dm.pool, slots)
    b.insert_frames(dm.pool, slots)
    ka, ca, wa, na = (x.cpu().numpy() for x in a.extract())
    kb, cb, wb, nb = (x.cpu().numpy() for x in b.extract())
    np.testing.assert_array_equal(ka, kb)
    np.testing.assert_array_equal(na, nb)
    # binned in-voxel offsets are quantised to cell/256: <= cell/512 = 39 um
    assert np.max(np.abs(ca - cb)) < 0.02 / 512 + 2e-6
    np.testing.assert_allclose(wa, wb, rtol=1e-5)


def test_binned_points_and_partials_roundtrip(binned, monkeypatch):
    """insert_points (exact float64 transform) far from the origin, then the
    owner-bucketed partials merged into block-hash owner maps reproduce the
    map (the multi-GPU exchange path, dist.MapExchange)."""
    from paper_2510_02080_b200 import _lib, dist as pdist, mapping
    rng = np.random.default_rng(3)
    x = rng.uniform(-1.0, 1.0, size=(200000, 3)) + np.array([1234.5, -987.25, 20.0])
    conf = rng.uniform(0.0, 1.0, size=len(x))
    conf[rng.random(len(x)) < 0.05] = 0.0
    vm = mapping.VoxelMap(0.02, 1 << 21)
    vm.insert_points(torch.as_tensor(x, device="cuda"), torch.as_tensor(conf, device="cuda"),
                     [1.0, 1.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0])
    k0, c0, w0, n0 = (t.cpu().numpy() for t in vm.extract())
    o = ofuse.fuse_points(x, conf, 0.02)
    np.testing.assert_array_equal(k0, o["keys"])
    np.testing.assert_array_equal(n0, o["count"])
    assert np.max(np.abs(c0 - o["centroid"])) < 1e-3  # float32 output at 1.2 km
    np.testing.assert_allclose(w0, o["wsum"], rtol=1e-5, atol=1e-8)  # fixed point: 2^-32 per term
    U = len(k0)
    L = _lib.lib()
    monkeypatch.delenv("EC3R_FUSE_ENGINE")  # owner maps merge into the block hash
    for n_ranks in (1, 3):
        keys = torch.empty(U, dtype=torch.int64, device="cuda")
        sums = torch.empty((U, 4), dtype=torch.float32, device="cuda")
        cnt = torch.empty(U, dtype=torch.int32, device="cuda")
        rc = torch.zeros(n_ranks, dtype=torch.int64, device="cuda")
        ws = torch.empty(L.ec3r_vhash_extract_workspace(vm.handle) + 1024, dtype=torch.uint8, device="cuda")
        _lib.check(L.ec3r_vhash_extract_partials(vm.handle, n_ranks, _lib.ptr(keys), _lib.ptr(sums), _lib.ptr(cnt),
                                                 _lib.ptr(rc), _lib.ptr(ws), ws.numel(), None), "partials")
        rcn = rc.cpu().numpy()
        assert rcn.sum() == U
        kn = keys.cpu().numpy()
        off = np.concatenate([[0], np.cumsum(rcn)])
        for r in range(n_ranks):
            assert np.all(pdist.owner_of(kn[off[r]:off[r + 1]], n_ranks) == r)
        merged = mapping.VoxelMap(0.02, 1 << 21)
        _lib.check(L.ec3r_vhash_merge_partials(merged.handle, _lib.ptr(keys), _lib.ptr(sums), _lib.ptr(cnt), U,
                                               None), "merge")
        k1, c1, w1, n1 = (t.cpu().numpy() for t in merged.extract())
        np.testing.assert_array_equal(k1, k0)
        np.testing.assert_array_equal(n1, n0)
        np.testing.assert_allclose(w1, w0, rtol=1e-6)
        assert np.max(np.abs(c1 - c0)) < 1e-3  # float32 centroids at 1.2 km


def test_tma_strip_insert_vs_oracle(golden, monkeypatch):
    """The opt-in TMA strip form of the block-hash insert (EC3R_FI_TMA=1:
    8-row strips of depth and confidence through a 2-stage cp.async.bulk
    ring) against the declared fusion rule, and equal keys / counts to the
    default register-loaded form on a full-resolution bench-generator map."""
    monkeypatch.setenv("EC3R_FI_TMA", "1")
    g = golden("mapping")
    dm, sms, sms_g = _registered(g)
    for cell in (0.02, 0.05):
        dm._vmap = None
        out = dm.fused_cloud(voxel=cell)
        o = ofuse.fuse_submaps(sms_g, _globs(sms), cell)
        np.testing.assert_array_equal(out["keys"], o["keys"])
        np.testing.assert_array_equal(out["count"], o["count"])
        np.testing.assert_allclose(out["wsum"], o["wsum"], rtol=1e-5)
        assert np.max(np.abs(out["centroid"] - o["centroid"])) < 1e-4
    from paper_2510_02080_b200 import mapping, synth
    cfg = synth.SceneConfig()
    sb = synth.make_submaps(31, cfg, seed=11, device="cuda")
    dm2 = mapping.DenseMapping(cfg.height, cfg.width, sb.K4)
    sms2 = [dm2.add_submap(ids, sb.depth[o:o + len(ids)], sb.conf[o:o + len(ids)], list(sb.poses8[o:o + len(ids)]))
            for ids, o in zip(sb.frame_ids, sb.slot_offsets)]
    dm2.register_chain(sms2)
    slots = torch.as_tensor(np.concatenate([sm.slots for sm in sms2]).astype(np.int32), device="cuda")
    _, a, _ = mapping.fuse_slots(dm2.pool, slots, 0.02)
    monkeypatch.delenv("EC3R_FI_TMA")
    _, b, _ = mapping.fuse_slots(dm2.pool, slots, 0.02)
    assert a[0].numel() > 100_000
    assert torch.equal(a[0], b[0]) and torch.equal(a[3], b[3])
    assert torch.allclose(a[2], b[2], rtol=1e-5)
    assert float((a[1] - b[1]).abs().max()) < 1e-5


def test_reduction_floor_diag_log_and_replay():
    """ec3r_vhash_diag_log / _replay (the bench's reduction-floor measure):
    the logged runs cover every fused point exactly once (their counts sum to
    n_points_in), the logging insert leaves the map unreduced, and replaying
    the log with counts reproduces the normal insert's voxel keys and counts."""
    from paper_2510_02080_b200 import _lib, mapping, synth
    cfg = synth.SceneConfig()
    sb = synth.make_submaps(11, cfg, seed=7, device="cuda")
    dm = mapping.DenseMapping(cfg.height, cfg.width, sb.K4)
    sms = [dm.add_submap(ids, sb.depth[o:o + len(ids)], sb.conf[o:o + len(ids)], list(sb.poses8[o:o + len(ids)]))
           for ids, o in zip(sb.frame_ids, sb.slot_offsets)]
    dm.register_chain(sms)
    slots = torch.as_tensor(np.concatenate([sm.slots for sm in sms]).astype(np.int32), device="cuda")
    vm, ref_out, st = mapping.fuse_slots(dm.pool, slots, 0.02)
    L = _lib.lib()
    cap = int(slots.numel()) * cfg.height * cfg.width
    runs = torch.empty((cap, 2), dtype=torch.int32, device="cuda")
    n_dev = torch.zeros(1, dtype=torch.int64, device="cuda")
    vm.clear()
    _lib.check(L.ec3r_vhash_diag_log(vm._h, _lib.ptr(runs), cap, _lib.ptr(n_dev)), "diag_log")
    vm.insert_frames(dm.pool, slots)
    n = int(n_dev.item())
    assert 0 < n <= st["n_points_in"]
    assert int(runs[:n, 1].sum().item()) == st["n_points_in"]
    assert vm.count() == 0  # logged, not reduced
    _lib.check(L.ec3r_vhash_diag_replay(vm._h, _lib.ptr(runs), _lib.ptr(n_dev), cap, 1, None), "diag_replay")
    keys, _, _, cnt = vm.extract(sort=True)
    assert torch.equal(keys, ref_out[0]) and torch.equal(cnt, ref_out[3])
