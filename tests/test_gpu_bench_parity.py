"""Parity at the bench configurations (BASELINE configs[1] and configs[3]):
the exact bench.Step of the headline number is run on the device and every
output is checked against the CPU oracle (oracle/, the reference's
algorithm restated and pinned to its golden vectors):

  * every registration edge (mapping.py:162-188, registration.py:38-102):
    status and keep count bit-exact, Sim(3) within 1e-5 relative;
  * every chained global pose (mapping.py:190-211: strongest partner,
    left fold of compositions) within 1e-5 relative;
  * the full fused map (mapping.py:56-57,332-338 + the declared voxel rule,
    oracle/fuse.py) at 2 cm: keys and counts bit-exact, centroids within
    1e-4 m, wsum within 1e-4 relative;
  * a 5 % sample of the step's 1500 tracking matches (tracking.py:143-170)
    bit-exact;
  * configs[3] global retrieval at K = 1,500 and 4,000 (loops.py:184-243):
    admitted pairs bit-exact and in the reference's emission order.
"""

import os
import sys

import numpy as np
import pytest
import torch

from oracle import fuse as ofuse
from oracle import ref_numpy as ref

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
SIM3_RTOL = 1e-5
# device status codes (include/ec3r_b200.h EC3R_ST_*) -> oracle status strings
ST = {0: ref.STATUS_OK, 1: ref.STATUS_SKIP, 2: ref.STATUS_TOO_FEW, 3: ref.STATUS_ALL_ZERO, 4: ref.STATUS_DEGENERATE,
      5: ref.STATUS_DEGENERATE}


@pytest.fixture(scope="module")
def bench_step():
    if not torch.cuda.is_available():
        pytest.skip("needs CUDA")
    import bench

    dm, sms, desc, halo = bench.build_workload(0, 1, 300, 1024, "cuda")
    step = bench.Step(dm, sms, desc, halo=halo)
    step.run()  # sizes the voxel map (outside the timed region in bench.py)
    step.run()
    out = tuple(x.clone() for x in step.run())
    torch.cuda.synchronize()
    if step.n_dev is not None:  # the step's host-sync-free emit: U only on the device
        assert int(step.n_dev.item()) == int(out[0].shape[0])
    reg = step.plan.run(dm.pool)
    torch.cuda.synchronize()
    dense = []
    for sm in sms:
        sl = torch.as_tensor(np.asarray(sm.slots, np.int64), device="cuda")
        p8 = dm.pool.poses[sl].cpu().numpy()
        dense.append(dict(depth=dm.pool.depth[sl].cpu().numpy(), conf=dm.pool.conf[sl].cpu().numpy(),
                          frame_ids=np.array(sm.keyframe_ids), pose_q=p8[:, 1:5], pose_t=p8[:, 5:],
                          K=np.asarray(dm.pool.K4)))
    return dict(step=step, sms=sms, out=out, reg=tuple(x.cpu().numpy() for x in reg), dense=dense, desc=desc)


def _sim3_close(v, s, q, t):
    assert abs(v[0] - s) <= SIM3_RTOL * abs(s), (v[0], s)
    np.testing.assert_allclose(ref.canonical_quat(v[1:5]), ref.canonical_quat(q), atol=SIM3_RTOL)
    np.testing.assert_allclose(v[5:], t, atol=SIM3_RTOL * max(1.0, float(np.abs(t).max())))


def test_bench_registration_edges_vs_oracle(bench_step):
    step, dense = bench_step["step"], bench_step["dense"]
    sim3, rms, count, npairs, status = bench_step["reg"][:5]
    index = {sm.id: i for i, sm in enumerate(bench_step["sms"])}
    assert len(step.plan.pairs) >= 58
    for e, (a, b) in enumerate(step.plan.pairs):
        o = ref.registration_edge(dense[index[a.id]], dense[index[b.id]])
        assert ST[int(status[e])] == o["status"], (e, int(status[e]), o["status"])
        assert int(npairs[e]) == o["n_pairs"], e
        if int(status[e]) == 0:
            assert int(count[e]) == o["count"], e  # confidence-floor keep mask bit-exact (its popcount)
            _sim3_close(sim3[e], o["s"], o["q"], o["t"])
            assert abs(rms[e] - o["rms"]) <= 1e-5 * max(o["rms"], 1e-9)


def test_bench_chained_poses_vs_oracle(bench_step):
    """Every submap's global pose: the oracle's edges chained on the host in
    registration order (left fold, strongest partner = max count, first on
    ties), against the device chain (pointer jumping)."""
    step, dense, sms = bench_step["step"], bench_step["dense"], bench_step["sms"]
    sub_g, sub_st = bench_step["reg"][5], bench_step["reg"][6]
    index = {sm.id: i for i, sm in enumerate(sms)}
    best = {}
    for e, (a, b) in enumerate(step.plan.pairs):
        o = ref.registration_edge(dense[index[a.id]], dense[index[b.id]])
        if o["status"] == ref.STATUS_OK:
            j = index[a.id]
            if j not in best or o["count"] > best[j][0]:
                best[j] = (o["count"], index[b.id], (o["s"], o["q"], o["t"]))
    glob = {0: (1.0, np.array([1.0, 0, 0, 0]), np.zeros(3))}
    for j in range(1, len(sms)):
        _, p, tr = best[j]
        glob[j] = ref.sim3_compose(glob[p], tr)
    assert (sub_st == 0).all()
    for j in range(len(sms)):
        s, q, t = glob[j]
        _sim3_close(sub_g[j], s, q, t)


def test_bench_fused_map_vs_oracle(bench_step):
    """The full configs[1] map (~3.8 M voxels at 2 cm from ~72 M points),
    fused by the oracle from the same decoded planes under the device's
    chained poses: the fusion stage is compared on identical inputs."""
    dense, sub_g = bench_step["dense"], bench_step["reg"][5]
    keys, cen, wsum, cnt = (x.cpu().numpy() for x in bench_step["out"])
    globs = [(float(v[0]), v[1:5], v[5:]) for v in sub_g]
    o = ofuse.fuse_submaps(dense, globs, 0.02)
    assert len(o["keys"]) > 3_000_000
    np.testing.assert_array_equal(keys, o["keys"])
    np.testing.assert_array_equal(cnt, o["count"])
    assert np.max(np.abs(cen - o["centroid"])) < 1e-4
    np.testing.assert_allclose(wsum, o["wsum"], rtol=1e-4)


def test_bench_tracking_matches_sample_vs_oracle(bench_step):
    """Every 20th of the 1500 tracked frames (5 %): the step's matches (each
    frame against its keyframe interval's resident map) bit-exact."""
    step = bench_step["step"]
    A, B, a_off, b_off, b_row = bench_step["desc"]
    mb = step.mb.cpu().numpy()
    a = A.view(torch.bfloat16)
    b = B.view(torch.bfloat16)
    n_frames = len(a_off) - 1
    checked = 0
    for f in range(0, n_frames, 20):
        fa = a[a_off[f]:a_off[f + 1]].double().cpu().numpy()
        M = int(b_off[f + 1] - b_off[f])
        fb = b[b_row[f]:b_row[f] + M].double().cpu().numpy()
        exp = ref.match_descriptors_vec(fa, fb, 0.8)
        seg = mb[a_off[f]:a_off[f + 1]]
        ia = np.flatnonzero(seg >= 0)
        np.testing.assert_array_equal(np.stack([ia, seg[ia]], axis=1), exp, err_msg=f"frame {f}")
        checked += 1
    assert checked >= 75


@pytest.mark.parametrize("K", [1500, 4000])
def test_configs3_retrieval_vs_oracle(K):
    """configs[3] / configs[4] databases: update_similarity's admitted list
    (two calls: admitted-once state) equals the oracle's."""
    if not torch.cuda.is_available():
        pytest.skip("needs CUDA")
    from paper_2510_02080_b200 import loops, synth
    pooled = synth.pooled_embeddings(K, device="cpu").numpy()
    kfs = np.arange(K, dtype=np.int64) * 2 + 1
    db = loops.RetrievalDB(pooled.shape[1], 1024)
    db.append(kfs, pooled)

    class Cfg:
        tau_global, tau_local = 0.93, 0.96

        @staticmethod
        def exclusion_zone():
            return 15

    mat = loops.SimilarityMatrix()
    st = ref.SimilarityState()
    for call in range(2):
        got = db.update(mat, 5, Cfg)
        exp = ref.update_similarity(st, kfs, pooled, 5, 15, 0.93, 0.96)
        assert [p for p, _ in got] == [p for p, _ in exp], call
        np.testing.assert_allclose([s for _, s in got], [s for _, s in exp], rtol=0, atol=1e-14)
    assert len(st.admitted) > 1000


def test_bench_step_run_to_run_determinism(bench_step):
    """the same step twice gives bit-identical registration
    (fixed-order cluster reductions), pose chain, tracking matches and voxel
    keys / counts (the block-hash float sums may differ in the last bits:
    atomics; the binned engine's integer sums are bit-exact, see
    test_gpu_fusion_engines)."""
    step = bench_step["step"]
    out2 = tuple(x.clone() for x in step.run())
    mb2 = step.mb.clone()
    torch.cuda.synchronize()
    reg2 = tuple(x.cpu().numpy() for x in step.plan.run(step.dm.pool))
    for a, b in zip(bench_step["reg"], reg2):
        np.testing.assert_array_equal(a, b)
    out1 = bench_step["out"]
    assert torch.equal(out1[0], out2[0]) and torch.equal(out1[3], out2[3])
    assert float((out1[1] - out2[1]).abs().max()) < 1e-6
    mb3 = step.mb.clone()
    step.run()
    assert torch.equal(mb2, mb3) and torch.equal(mb2, step.mb)
