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


def _build(ids_sel=None, id0=None):
    from paper_2510_02080_b200 import mapping, synth
    cfg = synth.SceneConfig()
    sb = synth.make_submaps(N_KF, cfg, seed=SEED, device="cuda")
    dm = mapping.DenseMapping(cfg.height, cfg.width, sb.K4)
    if id0 is not None:
        dm._next_id = id0  # global submap ids: windows number from their first index
    idx = range(len(sb.frame_ids)) if ids_sel is None else ids_sel
    sms = []
    for i in idx:
        ids, o = sb.frame_ids[i], sb.slot_offsets[i]
        sms.append(dm.add_submap(ids, sb.depth[o:o + len(ids)], sb.conf[o:o + len(ids)],
                                 list(sb.poses8[o:o + len(ids)])))
    return dm, sms, len(sb.frame_ids)


def _init(rank, world, port, backend):
    """gloo (CUDA payloads staged through the host) or NCCL itself: two NCCL
    ranks on one GPU take distinct NCCL_HOSTIDs (NCCL then treats them as
    separate hosts and uses its socket transport on loopback; validation of
    the NCCL forms, not a measurement)."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    if backend == "nccl":
        os.environ.update(NCCL_HOSTID=f"ec3r-test-rank{rank}", NCCL_SOCKET_IFNAME="lo", NCCL_IB_DISABLE="1")
        torch.cuda.set_device(0)
        dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", 0))
    else:
        dist.init_process_group("gloo", rank=rank, world_size=world)


def _poses(sms):
    from paper_2510_02080_b200.types import sim3_to_vec
    return np.stack([sim3_to_vec(sm.global_pose) for sm in sms])


def _worker(rank, world, port, q, backend="gloo"):
    _init(rank, world, port, backend)
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


@pytest.mark.parametrize("backend", ["gloo", "nccl"])
def test_register_window_two_ranks_equals_single_process(backend):
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, backend)) for r in range(world)]
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


def _chain_worker(rank, world, port, q, backend="gloo"):
    _init(rank, world, port, backend)
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


@pytest.mark.parametrize("backend", ["gloo", "nccl"])
def test_window_chain_device_two_ranks_equals_single_chain(backend):
    """The bench's N > 1 registration step (dist.WindowChain: halo P2P,
    ChainPlan, all-gather of window poses, ec3r_apply_window_offset) on two
    ranks equals the single-process device chain over the whole sequence."""
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_chain_worker, args=(r, world, port, q, backend)) for r in range(world)]
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


def _ret_worker(rank, world, port, q, backend="gloo"):
    _init(rank, world, port, backend)
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


@pytest.mark.parametrize("backend", ["gloo", "nccl"])
def test_retrieval_sharded_two_ranks_equals_single_and_oracle(backend):
    """dist.retrieval_sharded with two ranks (gloo, one GPU): each rank scores
    its coarse rows on the device; the gathered lists equal the single-GPU
    lists, and the admitted pairs equal the oracle's update_similarity."""
    from oracle import ref_numpy as ref
    from paper_2510_02080_b200 import loops, synth
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_ret_worker, args=(r, 2, port, q, backend)) for r in range(2)]
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


# -- loop edges across shards + pose-graph data path + the host-sync-free map
#    exchange --------------------------------------------------

LOOP_ID = 100


def _loop_frames(sb, kf_a, kf_b):
    """A loop submap over keyframes kf_a, kf_b (mapping.py:282-318): planes
    and local poses of their first decoded copies, re-anchored at kf_a."""
    out = []
    for kf in (kf_a, kf_b):
        for i, ids in enumerate(sb.frame_ids):
            if kf in ids:
                o = sb.slot_offsets[i] + list(ids).index(kf)
                out.append((sb.depth[o], sb.conf[o], np.asarray(sb.poses8[o])))
                break
    return out


def _loop_worker(rank, world, port, q, backend="gloo"):
    _init(rank, world, port, backend)
    try:
        from paper_2510_02080_b200 import dist as D
        from paper_2510_02080_b200 import mapping, synth
        torch.cuda.set_device(0)
        cfg = synth.SceneConfig()
        sb = synth.make_submaps(N_KF, cfg, seed=SEED, device="cuda")
        S = len(sb.frame_ids)
        lo, hi = D.shard_window(S, world, rank)
        dm, sms, _ = _build(range(lo, hi), id0=lo)
        D.register_window(dm, sms)
        directory = D.SubmapDirectory(dm)
        loop_sm = None
        kf_a, kf_b = sb.frame_ids[1][2], sb.frame_ids[S - 2][3]  # on rank 0 and rank 1
        if rank == world - 1:
            fr = _loop_frames(sb, kf_a, kf_b)
            dm._next_id = LOOP_ID
            loop_sm = dm.add_submap([kf_a, kf_b], torch.stack([f[0] for f in fr]), torch.stack([f[1] for f in fr]),
                                    [f[2] for f in fr])
        edges = D.register_loop_sharded(dm, loop_sm, directory)
        loop_pose = None if loop_sm is None else D.edge_rows([(0, 0, loop_sm.global_pose, 1.0)])[0][2:10]
        all_edges = [e[:4] for e in dm.edges]
        try:
            fn = D.reference_pgo()
        except ImportError:
            fn = None
        pgo = D.optimize_sharded(dm, all_edges, fn) if fn is not None else None
        # host-sync-free owner-partitioned map exchange
        slots = dm.all_slots()
        local, out, _ = mapping.fuse_slots(dm.pool, slots, 0.02)
        ex = D.MapExchange(0.02)
        a = ex.run(local, int(out[0].shape[0]), sync=False)
        ex.verify()
        n = int(a[4].item())
        a = tuple(x.clone() for x in a)
        cap0 = ex.cap
        cap1 = ex.retune()  # slabs sized from the observed buckets: same partition
        a2 = ex.run(local, int(out[0].shape[0]), sync=False)
        ex.verify()
        assert cap1 < cap0 and int(a2[4].item()) == n
        assert all(torch.equal(x[:n], y[:n]) for x, y in zip(a[:4], a2[:4]))
        b = D.MapExchange(0.02).run(local, int(out[0].shape[0]))
        res = dict(edges=[(i, j, D.edge_rows([(i, j, t, inf)])[0], c, r) for i, j, t, inf, c, r in edges],
                   loop=loop_pose,
                   pgo=pgo, async_map=tuple(x[:n].cpu().numpy() for x in a[:4]),
                   sync_map=tuple(x.cpu().numpy() for x in b), n_edges=len(all_edges),
                   final={sid: D.edge_rows([(0, 0, sm.global_pose, 1.0)])[0][2:10] for sid, sm in dm.submaps.items()})
        q.put((rank, res))
    except Exception as e:  # surface the failure in the parent
        import traceback
        q.put((rank, RuntimeError(traceback.format_exc())))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("backend", ["gloo", "nccl"])
def test_loop_edges_across_shards_pgo_and_map_exchange(backend):
    """Two ranks (gloo, one GPU): a loop submap on rank 1 sharing keyframes
    with a submap of each rank is registered through dist.fetch_frames +
    one batched launch; its edges and pose equal single-process registration
    (mapping.py:282-318).  optimize_sharded gathers every node and edge to
    rank 0, runs the reference's PoseGraph and broadcasts: equal to the
    single-process graph.  The fixed-slab MapExchange (no host round trip)
    gives, over both ranks, the single-process fused map."""
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_loop_worker, args=(r, world, port, q, backend)) for r in range(world)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=600) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    for v in out.values():
        if isinstance(v, Exception):
            raise v
    from oracle import ref_numpy as ref
    from paper_2510_02080_b200 import dist as D
    from paper_2510_02080_b200 import synth
    # single process: the whole sequence, then the same loop submap
    dm, sms, S = _build()
    dm.register_chain(sms)
    cfg = synth.SceneConfig()
    sb = synth.make_submaps(N_KF, cfg, seed=SEED, device="cuda")
    kf_a, kf_b = sb.frame_ids[1][2], sb.frame_ids[S - 2][3]
    fr = _loop_frames(sb, kf_a, kf_b)
    dm._next_id = LOOP_ID
    loop_sm = dm.add_submap([kf_a, kf_b], torch.stack([f[0] for f in fr]), torch.stack([f[1] for f in fr]),
                            [f[2] for f in fr])
    edges = dm.registration_edges(loop_sm)
    best = max(edges, key=lambda e: e[3])
    loop_sm.global_pose = dm.submaps[best[0]].global_pose.compose(best[1])
    got = out[world - 1]
    assert [e[0] for e in got["edges"]] == [e[0] for e in edges] and len(edges) == 2
    assert {e[0] for e in edges} == {1, S - 2}  # one partner on each shard
    for (gi, gj, row, c, r), (sid, tr, info, count, rms) in zip(got["edges"], edges):
        assert gj == LOOP_ID and c == count  # keep counts bit-exact
        exp = D.edge_rows([(sid, LOOP_ID, tr, info)])[0]
        assert abs(row[2] - exp[2]) <= 1e-9 * exp[2]
        np.testing.assert_allclose(ref.canonical_quat(row[3:7]), ref.canonical_quat(exp[3:7]), atol=1e-9)
        np.testing.assert_allclose(row[7:10], exp[7:10], atol=1e-9)
        assert abs(r - rms) <= 1e-9 * max(rms, 1e-9)
    exp_loop = D.edge_rows([(0, 0, loop_sm.global_pose, 1.0)])[0][2:10]
    np.testing.assert_allclose(got["loop"][5:], exp_loop[5:], atol=1e-8)
    assert out[0]["loop"] is None and out[0]["edges"] == []
    # every edge of the single-process graph is gathered exactly once
    assert sum(out[r]["n_edges"] for r in range(world)) == len(dm.edges) + len(edges)
    for e in edges:
        dm.edges.append((e[0], LOOP_ID, e[1], e[2]))
    dm._commit(loop_sm)
    if out[0]["pgo"] is not None:
        nodes = {sid: D.edge_rows([(0, 0, sm.global_pose, 1.0)])[0][2:10] for sid, sm in dm.submaps.items()}
        exp = D.reference_pgo()(nodes, D.edge_rows(dm.edges))
        assert sorted(exp) == sorted(out[0]["pgo"])
        for r in range(world):
            for sid, v in exp.items():  # inputs agree to ~1e-12 (window prefix composition order)
                np.testing.assert_allclose(out[r]["pgo"][sid], v, atol=1e-7)
    # owner-partitioned map: both ranks' partitions = the single-process map
    # under the ranks' final (post-PGO) poses
    from paper_2510_02080_b200.types import vec_to_sim3
    for r in range(world):
        for sid, v in out[r]["final"].items():
            dm.submaps[sid].global_pose = vec_to_sim3(v)
            dm._commit(dm.submaps[sid])
    ref_map = dm.fused_cloud(voxel=0.02)
    for mode in ("async_map", "sync_map"):
        keys = np.concatenate([out[r][mode][0] for r in range(world)])
        cnt = np.concatenate([out[r][mode][3] for r in range(world)])
        assert len(np.unique(keys)) == len(keys)  # owners are disjoint
        order = np.argsort(keys)
        for r in range(world):
            k = out[r][mode][0]
            assert np.all(np.diff(k) > 0)  # each partition sorted
            np.testing.assert_array_equal(D.owner_of(k, world), r)
        np.testing.assert_array_equal(keys[order], ref_map["keys"])
        np.testing.assert_array_equal(cnt[order], ref_map["count"])
    for r in range(world):
        for a, b in zip(out[r]["async_map"], out[r]["sync_map"]):
            np.testing.assert_array_equal(a, b)
