"""Multi-process (gloo, world_size 2, CPU) tests of the N>1 host protocol:
window sharding, ragged all-gather, the owner-bucketed all-to-all of voxel
partials and the owner-side merge, checked against the single-process oracle
fusion (oracle/fuse.py).  The device halves of the protocol
(ec3r_vhash_extract_partials / merge_partials) are covered by the GPU tests."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import fuse as ofuse
from paper_2510_02080_b200 import dist as D

WORLD = 2
CELL = 0.02


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, fn_name, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        q.put((rank, globals()[fn_name](rank, world)))
    except Exception as e:  # surface the failure in the parent
        q.put((rank, e))
    finally:
        dist.destroy_process_group()


def _spawn(fn_name, world=WORLD):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, fn_name, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = {}
    for _ in range(world):
        r, v = q.get(timeout=120)
        out[r] = v
    for p in procs:
        p.join(timeout=60)
    for r, v in out.items():
        if isinstance(v, Exception):
            raise v
    return out


# ---------------------------------------------------------------------------
# helpers shared by the workers (module level: picklable under spawn)

def _points(seed, n=20000):
    rng = np.random.default_rng(seed)
    x = rng.uniform(-0.3, 0.3, size=(n, 3))
    conf = rng.uniform(0.05, 1.0, size=n)
    conf[rng.random(n) < 0.05] = 0.0  # dropped by rule (ii)
    return x, conf


def _local_partials(x, conf, world):
    """What one rank's device hash holds after fusing its own points, as the
    raw partials ec3r_vhash_extract_partials emits: (key, sum c*(x - corner),
    sum c, count) bucketed by owner rank."""
    live = conf > 0
    x, conf = x[live], conf[live]
    cells = ofuse.voxel_cells(x, CELL)
    from oracle.ref_numpy import pack
    keys = pack(cells)
    uniq, inv = np.unique(keys, return_inverse=True)
    corner = cells * CELL
    s = np.zeros((len(uniq), 4))
    np.add.at(s[:, :3], inv, conf[:, None] * (x - corner))
    np.add.at(s[:, 3], inv, conf)
    cnt = np.bincount(inv, minlength=len(uniq)).astype(np.int32)
    own = D.owner_of(uniq, world)
    order = np.argsort(own, kind="stable")
    rank_counts = np.bincount(own, minlength=world)
    return uniq[order].astype(np.int64), s[order].astype(np.float32), cnt[order], rank_counts


def _merge(keys, sums4, cnt):
    uniq, inv = np.unique(keys, return_inverse=True)
    s = np.zeros((len(uniq), 4))
    np.add.at(s, inv, sums4.astype(np.float64))
    c = np.bincount(inv, weights=cnt, minlength=len(uniq)).astype(np.int64)
    return uniq, s, c


# ---------------------------------------------------------------------------
# workers

def w_exchange(rank, world):
    rng = np.random.default_rng(rank)
    n = 1000 + 337 * rank
    keys = rng.integers(0, 1 << 62, size=n, dtype=np.int64)
    sums = rng.standard_normal((n, 4)).astype(np.float32)
    cnt = rng.integers(1, 50, size=n).astype(np.int32)
    own = D.owner_of(keys, world)
    order = np.argsort(own, kind="stable")
    rc = np.bincount(own, minlength=world)
    k, s, c = D.exchange_partials(torch.as_tensor(keys[order]), torch.as_tensor(sums[order]),
                                  torch.as_tensor(cnt[order]), rc.tolist())
    return k.numpy(), s.numpy(), c.numpy()


def w_global_fusion(rank, world):
    x, conf = _points(7, 30000)
    lo, hi = D.shard_window(len(x), world, rank)
    keys, sums4, cnt, rc = _local_partials(x[lo:hi], conf[lo:hi], world)
    k, s, c = D.exchange_partials(torch.as_tensor(keys), torch.as_tensor(sums4), torch.as_tensor(cnt),
                                  rc.tolist())
    return _merge(k.numpy(), s.numpy(), c.numpy())


def w_gather(rank, world):
    t = torch.arange(3 + 4 * rank, dtype=torch.int64) + 100 * rank
    return [g.numpy() for g in D.gather_ragged(t)]


# ---------------------------------------------------------------------------
# tests

def test_shard_window_partitions():
    for n in (0, 1, 5, 59, 60, 61, 1000):
        for world in (1, 2, 3, 8):
            ws = [D.shard_window(n, world, r) for r in range(world)]
            assert ws[0][0] == 0 and ws[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(ws, ws[1:]))
            sizes = [b - a for a, b in ws]
            assert max(sizes) - min(sizes) <= 1


def test_owner_hash_matches_device_rule():
    # mix64 of csrc/vhash.cu (murmur3 finaliser) on known values
    k = np.array([0, 1, 2, (1 << 63) - 1], dtype=np.uint64)
    m = D.mix64(k)
    assert m[0] == 0
    ref = []
    for v in k.tolist():
        v ^= v >> 33
        v = (v * 0xFF51AFD7ED558CCD) & ((1 << 64) - 1)
        v ^= v >> 33
        v = (v * 0xC4CEB9FE1A85EC53) & ((1 << 64) - 1)
        v ^= v >> 33
        ref.append(v)
    assert m.tolist() == ref
    own = D.owner_of(np.arange(10000), 8)
    assert set(own.tolist()) == set(range(8))


def test_gather_ragged_gloo():
    out = _spawn("w_gather")
    for r in range(WORLD):
        got = out[r]
        assert len(got) == WORLD
        for src in range(WORLD):
            np.testing.assert_array_equal(got[src], np.arange(3 + 4 * src) + 100 * src)


def test_exchange_partials_routes_every_row_to_its_owner_gloo():
    out = _spawn("w_exchange")
    # reconstruct what every rank sent
    sent = []
    for r in range(WORLD):
        rng = np.random.default_rng(r)
        n = 1000 + 337 * r
        keys = rng.integers(0, 1 << 62, size=n, dtype=np.int64)
        sums = rng.standard_normal((n, 4)).astype(np.float32)
        cnt = rng.integers(1, 50, size=n).astype(np.int32)
        sent.append((keys, sums, cnt))
    for r in range(WORLD):
        k, s, c = out[r]
        assert np.all(D.owner_of(k, WORLD) == r)
        exp_k = np.concatenate([kk[D.owner_of(kk, WORLD) == r] for kk, _, _ in sent])
        exp_s = np.concatenate([ss[D.owner_of(kk, WORLD) == r] for kk, ss, _ in sent])
        exp_c = np.concatenate([cc[D.owner_of(kk, WORLD) == r] for kk, _, cc in sent])
        np.testing.assert_array_equal(k, exp_k)  # rank order, bucket order preserved
        np.testing.assert_array_equal(s, exp_s)
        np.testing.assert_array_equal(c, exp_c)


def test_global_fusion_protocol_equals_single_process_oracle_gloo():
    out = _spawn("w_global_fusion")
    x, conf = _points(7, 30000)
    ref = ofuse.fuse_points(x, conf, CELL)
    keys = np.concatenate([out[r][0] for r in range(WORLD)])
    sums = np.concatenate([out[r][1] for r in range(WORLD)])
    cnt = np.concatenate([out[r][2] for r in range(WORLD)])
    order = np.argsort(keys)
    keys, sums, cnt = keys[order], sums[order], cnt[order]
    # every voxel owned by exactly one rank, keys / counts bit-exact
    np.testing.assert_array_equal(keys, ref["keys"])
    np.testing.assert_array_equal(cnt, ref["count"])
    np.testing.assert_allclose(sums[:, 3], ref["wsum"], rtol=1e-5)
    from oracle.ref_numpy import unpack
    corner = unpack(keys).astype(np.float64) * CELL
    cen = corner + sums[:, :3] / sums[:, 3:4]
    assert np.max(np.abs(cen - ref["centroid"])) < 1e-4


# --------------------------------------------------------------------------
# align windows: halo exchange + prefix composition of window offsets

class _FakePool:
    def __init__(self, rank, n_frames=12, H=4, W=5):
        self.H, self.W, self.device = H, W, torch.device("cpu")
        g = torch.Generator().manual_seed(100 + rank)
        self.depth = torch.rand((n_frames, H, W), generator=g)
        self.conf = torch.rand((n_frames, H, W), generator=g)
        self.poses = torch.rand((n_frames, 8), generator=g, dtype=torch.float64)


class _FakeSubmap:
    def __init__(self, kf_ids, slots, sid=0):
        self.keyframe_ids, self.slots, self.id = tuple(kf_ids), np.asarray(slots), sid


class _FakeMapping:
    def __init__(self, rank):
        self.pool = _FakePool(rank)
        self.added = None
        self._next_id = 50

    def add_submap(self, ids, depth, conf, poses):
        self.added = (list(ids), depth.clone(), conf.clone(), np.stack(poses))
        sm = _FakeSubmap(ids, [], self._next_id)
        self._next_id += 1
        return sm


def _windows(rank):
    # flush order (new..., old): rank 0 = [(0..5), (6..10, 5)], rank 1 = [(11..15, 10), (16..20, 15)]
    if rank == 0:
        return [_FakeSubmap(range(6), range(6), 0), _FakeSubmap(list(range(6, 11)) + [5], range(6, 12), 1)]
    return [_FakeSubmap(list(range(11, 16)) + [10], range(6), 2),
            _FakeSubmap(list(range(16, 21)) + [15], range(6, 12), 3)]


def w_halo(rank, world):
    m = _FakeMapping(rank)
    stub = D.window_halo(m, _windows(rank))
    # the stub names the predecessor's submap (global id 1) and takes no id
    # of this rank's sequence
    assert stub is None or (stub.remote_id == 1 and stub.id < 0 and m._next_id == 50)
    return m.added


def _tf(rng):
    q = rng.normal(size=4)
    q /= np.linalg.norm(q)
    return np.concatenate([[rng.uniform(0.5, 2.0)], q, rng.normal(size=3)])


def w_offset(rank, world):
    rng = np.random.default_rng(rank)
    return D.window_offset(_tf(rng))


def test_window_halo_sends_the_shared_keyframe_frame_gloo():
    out = _spawn("w_halo")
    assert out[0] is None
    ids, depth, conf, poses = out[1]
    assert ids == [10]  # rank 1's first submap shares keyframe 10 with rank 0's last submap
    src = _FakePool(0)
    k = 4 + 6  # keyframe 10 is frame 4 of rank 0's last submap, pool slot 10
    np.testing.assert_array_equal(depth.numpy(), src.depth[k:k + 1].numpy())
    np.testing.assert_array_equal(conf.numpy(), src.conf[k:k + 1].numpy())
    np.testing.assert_array_equal(poses, src.poses[k:k + 1].numpy())


def test_window_offsets_prefix_compose_gloo():
    from paper_2510_02080_b200.types import vec_to_sim3
    out = _spawn("w_offset")
    w0 = _tf(np.random.default_rng(0))
    np.testing.assert_allclose(out[0], [1, 1, 0, 0, 0, 0, 0, 0], atol=0)
    exp = vec_to_sim3(D.prefix_offsets([w0, w0])[1])
    got = vec_to_sim3(out[1])
    assert abs(got.scale - vec_to_sim3(w0).scale) < 1e-15 and abs(exp.scale - got.scale) == 0
    np.testing.assert_allclose(got.translation, vec_to_sim3(w0).translation, atol=1e-15)


def test_prefix_offsets_compose_in_rank_order():
    """O_r = W_0 o ... o W_{r-1}: the global pose of window r's reference
    frame, for any number of windows (pure host math of window_offset)."""
    from paper_2510_02080_b200.types import Sim3Transform, sim3_to_vec, vec_to_sim3
    rng = np.random.default_rng(11)
    W = [_tf(rng) for _ in range(5)]
    offs = D.prefix_offsets(W)
    acc = Sim3Transform.identity()
    for r in range(5):
        got = vec_to_sim3(offs[r])
        assert abs(got.scale - acc.scale) <= 1e-12 * acc.scale
        np.testing.assert_allclose(got.translation, acc.translation, atol=1e-9)
        np.testing.assert_allclose(np.abs(np.dot(got.rotation.q, acc.rotation.q)), 1.0, atol=1e-12)
        acc = acc.compose(vec_to_sim3(W[r]))
    np.testing.assert_array_equal(offs[0], sim3_to_vec(Sim3Transform.identity()))


# --------------------------------------------------------------------------
# sharded retrieval (dist.retrieval_sharded): per-rank coarse rows, ragged
# all-gather in rank order == the single-process lists

def _shard_lists(P, stride, excl, tau_g, tau_l, kb, ke):
    """Test-side restatement of the six K6 lists for coarse rows [kb, ke)
    in the reference's emission order (loops.py:218-243)."""
    K = P.shape[0]
    Kc = (K + stride - 1) // stride
    cp, cs, qp, qs, ep, es = [], [], [], [], [], []
    for ai in range(kb, ke):
        for bi in range(ai + 1, Kc):
            a, b = ai * stride, bi * stride
            if abs(a - b) < excl:
                continue
            s = float(P[a] @ P[b])
            cp.append((a, b))
            cs.append(s)
            if s <= tau_g:
                continue
            for da in range(-(stride - 1), stride):
                for db in range(-(stride - 1), stride):
                    ia, ib = a + da, b + db
                    if 0 <= ia < K and 0 <= ib < K and abs(ia - ib) >= excl:
                        sn = float(P[ia] @ P[ib])
                        ep.append((ia, ib))
                        es.append(sn)
                        if sn > tau_l:
                            qp.append((ia, ib))
                            qs.append(sn)
    f = lambda p: np.asarray(p, np.int32).reshape(-1, 2)  # noqa: E731
    return f(cp), np.asarray(cs), f(qp), np.asarray(qs), f(ep), np.asarray(es)


def _retrieval_db(K=300):
    from paper_2510_02080_b200 import synth
    return synth.pooled_embeddings(K, device="cpu").numpy()


class _HostShardDB:
    """RetrievalDB stand-in whose score() is the restated lists (CPU)."""

    def __init__(self, P):
        self.P, self.n = P, P.shape[0]
        self.vec = torch.as_tensor(P)

    def score(self, stride, excl, tau_g, tau_l, kb, ke):
        return _shard_lists(self.P, stride, excl, tau_g, tau_l, kb, ke)


def w_retrieval(rank, world):
    db = _HostShardDB(_retrieval_db())
    return D.retrieval_sharded(db, 5, 15, 0.93, 0.96)


def test_retrieval_sharded_merge_equals_single_gloo():
    out = _spawn("w_retrieval")
    P = _retrieval_db()
    Kc = (P.shape[0] + 4) // 5
    exp = _shard_lists(P, 5, 15, 0.93, 0.96, 0, Kc)
    assert len(exp[2]) > 0 and len(exp[0]) > 0  # the case has candidates
    for r in range(WORLD):
        for got, want in zip(out[r], exp):
            np.testing.assert_array_equal(got, want)


# ---------------------------------------------------------------------------
# loop edges across shards + the pose-graph data path (dist.SubmapDirectory,
# fetch_frames, gather_graph, optimize_sharded): a CPU "mapping" with a frame
# pool on the host -- the registration launch itself is covered on the GPU
# (tests/test_gpu_dist.py)

class _Pool:
    def __init__(self, H, W):
        self.H, self.W, self.device = H, W, torch.device("cpu")
        self.depth = torch.zeros((0, H, W))
        self.conf = torch.zeros((0, H, W))
        self.poses = torch.zeros((0, 8), dtype=torch.float64)


class _Sub:
    def __init__(self, sid, kfs, slots, g):
        from paper_2510_02080_b200.types import vec_to_sim3
        self.id, self.keyframe_ids, self.slots = sid, tuple(kfs), np.asarray(slots)
        self.global_pose = vec_to_sim3(g)


class _Mapping:
    """Rank r owns submaps 10r .. 10r+2; submap i holds keyframes (3i, 3i+1,
    3i+2); frame planes encode (submap, keyframe) so the test can check who
    answered."""

    def __init__(self, rank, H=4, W=5):
        self.pool = _Pool(H, W)
        self.submaps, self.edges, self.committed = {}, [], []
        d, c, p = [], [], []
        for i in range(3):
            sid = 10 * rank + i
            kfs = [3 * sid, 3 * sid + 1, 3 * sid + 2]
            slots = list(range(len(d), len(d) + 3))
            for kf in kfs:
                d.append(torch.full((H, W), float(1000 * sid + kf)))
                c.append(torch.full((H, W), 0.5 + 0.01 * kf))
                p.append(torch.tensor([1.0, 1, 0, 0, 0, kf, sid, 0], dtype=torch.float64))
            g = np.array([1.0 + 0.1 * sid, 1, 0, 0, 0, sid, 0, 0])
            self.submaps[sid] = _Sub(sid, kfs, slots, g)
        self.pool.depth, self.pool.conf, self.pool.poses = torch.stack(d), torch.stack(c), torch.stack(p)

    def _commit(self, sm):
        self.committed.append(sm.id)


def w_directory_fetch(rank, world):
    m = _Mapping(rank)
    dr = D.SubmapDirectory(m)
    # each rank asks for one frame of every other rank's middle submap, plus one of its own
    req = [(10 * r + 1, 3 * (10 * r + 1) + 2) for r in range(world) if r != rank] + [(10 * rank, 3 * 10 * rank)]
    got = D.fetch_frames(m, req, dr)
    out = {}
    for (sid, kf), (dep, cf, pose, glob) in got.items():
        out[(sid, kf)] = (float(dep[0, 0]), float(cf[1, 2]), pose.tolist(), glob.tolist())
    return dr.owner, dr.partners([3, 31, 4]), out


def test_directory_and_fetch_frames_gloo():
    out = _spawn("w_directory_fetch")
    for rank, (owner, partners, got) in out.items():
        assert owner == {0: 0, 1: 0, 2: 0, 10: 1, 11: 1, 12: 1}
        assert partners == [1, 10]  # keyframes 3, 31 (submap 10 holds 30..32), 4 (submap 1): first-seen order
        for (sid, kf), (dep, cf, pose, glob) in got.items():
            assert dep == 1000 * sid + kf  # the owner's copy of that submap's frame
            assert abs(cf - (0.5 + 0.01 * kf)) < 1e-6
            assert pose[5] == kf and pose[6] == sid
            assert abs(glob[0] - (1.0 + 0.1 * sid)) < 1e-12 and glob[5] == sid
        assert len(got) == 2


def w_pgo_path(rank, world):
    from paper_2510_02080_b200.types import vec_to_sim3
    m = _Mapping(rank)
    info = np.eye(7) * (5.0 + rank)
    edges = [(10 * rank, 10 * rank + 1, vec_to_sim3([1.0, 1, 0, 0, 0, 0.5, 0, 0]), info)]
    seen = {}

    def fn(nodes, rows):  # a stand-in optimiser: shift every translation by the edge count
        seen["nodes"] = sorted(nodes)
        seen["rows"] = rows.copy()
        return {sid: np.concatenate([v[:5], v[5:] + len(rows)]) for sid, v in nodes.items()}

    res = D.optimize_sharded(m, edges, fn)
    return seen, {k: v.tolist() for k, v in res.items()}, sorted(m.committed), \
        {sid: float(sm.global_pose.translation[0]) for sid, sm in m.submaps.items()}


def test_pose_graph_gather_and_broadcast_gloo():
    out = _spawn("w_pgo_path")
    seen0 = out[0][0]
    assert seen0["nodes"] == [0, 1, 2, 10, 11, 12]
    rows = seen0["rows"]
    assert rows.shape == (2, D.EDGE_COLS)
    assert rows[:, :2].tolist() == [[0, 1], [10, 11]]
    assert rows[:, 10].tolist() == [5.0, 6.0]
    assert out[1][0] == {}  # only the root runs the optimiser
    for rank, (_, res, committed, tx) in out.items():
        assert sorted(res) == [0, 1, 2, 10, 11, 12]
        assert committed == [10 * rank, 10 * rank + 1, 10 * rank + 2]  # own submaps re-committed
        for sid, x in tx.items():
            assert x == sid + 2  # translation x = sid, shifted by the 2 gathered edges
