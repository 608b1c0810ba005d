"""Two ranks on one GPU (gloo, CUDA payloads staged through the host) running
the sharded align protocol end to end: each rank registers its own window of
full-resolution synthetic submaps plus the predecessor's shared-frame halo
(dist.register_window); the resulting global poses must equal single-process
registration of the whole sequence, and the fused map of the two windows the
single-process fused map."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

N_KF = 31  # 6 submaps of 6 frames
SEED = 4


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _build(ids_sel=None):
    from paper_2510_02080_b200 import mapping, synth
    cfg = synth.SceneConfig()
    sb = synth.make_submaps(N_KF, cfg, seed=SEED, device="cuda")
    dm = mapping.DenseMapping(cfg.height, cfg.width, sb.K4)
    idx = range(len(sb.frame_ids)) if ids_sel is None else ids_sel
    sms = []
    for i in idx:
        ids, o = sb.frame_ids[i], sb.slot_offsets[i]
        sms.append(dm.add_submap(ids, sb.depth[o:o + len(ids)], sb.conf[o:o + len(ids)],
                                 list(sb.poses8[o:o + len(ids)])))
    return dm, sms, len(sb.frame_ids)


def _poses(sms):
    from paper_2510_02080_b200.types import sim3_to_vec
    return np.stack([sim3_to_vec(sm.global_pose) for sm in sms])


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2510_02080_b200 import dist as D
        torch.cuda.set_device(0)
        from paper_2510_02080_b200 import synth
        S = len(synth.flush_batches(N_KF))
        lo, hi = D.shard_window(S, world, rank)
        dm, sms, _ = _build(range(lo, hi))
        D.register_window(dm, sms)
        cloud = dm.fused_cloud(voxel=0.02)
        q.put((rank, (lo, hi, _poses(sms), len(dm.submaps), cloud["keys"], cloud["count"])))
    except Exception as e:  # surface the failure in the parent
        q.put((rank, e))
    finally:
        dist.destroy_process_group()


def test_register_window_two_ranks_equals_single_process():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = {}
    for _ in range(world):
        r, v = q.get(timeout=240)
        out[r] = v
    for p in procs:
        p.join(timeout=60)
    for v in out.values():
        if isinstance(v, Exception):
            raise v
    dm, sms, S = _build()
    dm.register_chain(sms)
    full = _poses(sms)
    from oracle import ref_numpy as ref
    for r in range(world):
        lo, hi, poses, n_sub, _, _ = out[r]
        assert n_sub == hi - lo  # the halo stub is not part of the map
        for j in range(lo, hi):
            a, b = poses[j - lo], full[j]
            assert abs(a[0] - b[0]) <= 1e-9 * b[0]
            np.testing.assert_allclose(ref.canonical_quat(a[1:5]), ref.canonical_quat(b[1:5]), atol=1e-9)
            np.testing.assert_allclose(a[5:], b[5:], atol=1e-9 * max(1.0, float(np.abs(b[5:]).max())))
    # the union of the windows' voxel maps covers the single-process map
    ref_map = dm.fused_cloud(voxel=0.02)
    keys = np.unique(np.concatenate([out[r][4] for r in range(world)]))
    cnt = {}
    for r in range(world):
        for k, c in zip(out[r][4], out[r][5]):
            cnt[int(k)] = cnt.get(int(k), 0) + int(c)
    np.testing.assert_array_equal(keys, ref_map["keys"])
    assert sum(cnt.values()) == int(ref_map["count"].sum())


def _chain_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2510_02080_b200 import dist as D
        from paper_2510_02080_b200 import mapping, synth
        torch.cuda.set_device(0)
        cfg = synth.SceneConfig()
        sb = synth.make_submaps(N_KF, cfg, seed=SEED, device="cuda")
        S = len(sb.frame_ids)
        lo, hi = D.shard_window(S, world, rank)
        send_pos, recv_ids = D.halo_handshake(sb.frame_ids[lo], sb.frame_ids[hi - 1])
        dm = mapping.DenseMapping(cfg.height, cfg.width, sb.K4)
        stub = None
        if recv_ids:  # zero planes: the halo must fill them
            z = torch.zeros((len(recv_ids), cfg.height, cfg.width), dtype=torch.float32, device="cuda")
            stub = dm.add_submap(recv_ids, z, z, [np.array([1.0, 1, 0, 0, 0, 0, 0, 0])] * len(recv_ids))
        sms = []
        for i in range(lo, hi):
            ids, o = sb.frame_ids[i], sb.slot_offsets[i]
            sms.append(dm.add_submap(ids, sb.depth[o:o + len(ids)], sb.conf[o:o + len(ids)],
                                     list(sb.poses8[o:o + len(ids)])))
        wc = D.WindowChain(dm, stub, sms, send_pos)
        for _ in range(2):  # repeated steps give the same poses
            out = wc.run()
        torch.cuda.synchronize()
        sub_g = out[5].cpu().numpy()[(1 if stub is not None else 0):]
        slot_g = dm.pool.globals[int(sms[0].slots[0]):int(sms[-1].slots[-1]) + 1].cpu().numpy()
        q.put((rank, (lo, hi, sub_g, slot_g, [len(sm.slots) for sm in sms], (out[6].cpu().numpy() == 0).sum())))
    except Exception as e:  # surface the failure in the parent
        q.put((rank, e))
    finally:
        dist.destroy_process_group()


def test_window_chain_device_two_ranks_equals_single_chain():
    """The bench's N > 1 registration step (dist.WindowChain: halo P2P,
    ChainPlan, all-gather of window poses, ec3r_apply_window_offset) on two
    ranks equals the single-process device chain over the whole sequence."""
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_chain_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = {}
    for _ in range(world):
        r, v = q.get(timeout=240)
        out[r] = v
    for p in procs:
        p.join(timeout=60)
    for v in out.values():
        if isinstance(v, Exception):
            raise v
    from oracle import ref_numpy as ref
    from paper_2510_02080_b200 import mapping
    dm, sms, S = _build()
    full = mapping.ChainPlan(sms).run(dm.pool)[5].cpu().numpy()
    for r in range(world):
        lo, hi, sub_g, slot_g, lens, n_ok = out[r]
        assert n_ok >= hi - lo - (1 if r == 0 else 0)
        for j in range(lo, hi):
            a, b = sub_g[j - lo], full[j]
            assert abs(a[0] - b[0]) <= 1e-9 * b[0]
            np.testing.assert_allclose(ref.canonical_quat(a[1:5]), ref.canonical_quat(b[1:5]), atol=1e-9)
            np.testing.assert_allclose(a[5:], b[5:], atol=1e-9 * max(1.0, float(np.abs(b[5:]).max())))
        np.testing.assert_array_equal(slot_g, np.repeat(sub_g, lens, axis=0))


K_RET = 1200


def _ret_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2510_02080_b200 import dist as D
        from paper_2510_02080_b200 import loops, synth
        torch.cuda.set_device(0)
        pooled = synth.pooled_embeddings(K_RET, device="cpu").numpy()
        db = loops.RetrievalDB(pooled.shape[1], 256)
        db.append(np.arange(K_RET) * 3 + 7, pooled)
        q.put((rank, D.retrieval_sharded(db, 5, 15, 0.93, 0.96)))
    except Exception as e:
        q.put((rank, e))
    finally:
        dist.destroy_process_group()


def test_retrieval_sharded_two_ranks_equals_single_and_oracle():
    """dist.retrieval_sharded with two ranks (gloo, one GPU): each rank scores
    its coarse rows on the device; the gathered lists equal the single-GPU
    lists, and the admitted pairs equal the oracle's update_similarity."""
    from oracle import ref_numpy as ref
    from paper_2510_02080_b200 import loops, synth
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_ret_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=600) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
    for v in out.values():
        if isinstance(v, Exception):
            raise v
    pooled = synth.pooled_embeddings(K_RET, device="cpu").numpy()
    db = loops.RetrievalDB(pooled.shape[1], 256)
    kfs = np.arange(K_RET) * 3 + 7
    db.append(kfs, pooled)
    single = db.score(5, 15, 0.93, 0.96)
    for r in range(2):
        for a, b in zip(out[r], single):
            np.testing.assert_array_equal(a, b)
    mat = loops.SimilarityMatrix()
    got = loops.admit(mat, kfs, out[0][2], out[0][3])
    exp = ref.update_similarity(ref.SimilarityState(), kfs, pooled, 5, 15, 0.93, 0.96)
    assert [p for p, _ in got] == [p for p, _ in exp]
    assert len(got) > 0
