"""Multi-GPU plumbing of the path (one process per GPU, torch.distributed).

SURVEY.md §8(e) / DESIGN.md §5:

* align + fuse shard by contiguous submap windows (``shard_window``): edges
  are independent (mapping.py:171-183), so registration has no collective;
* the global voxel map is partitioned by voxel key: every rank fuses its own
  frames into a local hash, buckets the raw partial sums by owner rank
  (``owner_of`` = mix64(key) mod world, the same hash as the device
  partitioner in csrc/vhash.cu), exchanges them in one all-to-all
  (``exchange_partials``) and merges what it owns (``fuse_global``);
* the retrieval database shards by coarse keyframe rows; the per-shard
  candidate lists come back in reference emission order when concatenated in
  rank order (``retrieval_sharded``);
* the matcher is replicas only (independent frame pairs).

The exchange helpers take tensors on any device, so the protocol runs under
``gloo`` on CPU in the tests and under NCCL on the GPUs.
"""

from __future__ import annotations

import math
from typing import Optional, Sequence

import numpy as np
import torch
import torch.distributed as dist

_M1 = 0xFF51AFD7ED558CCD
_M2 = 0xC4CEB9FE1A85EC53


def _world(group) -> tuple[int, int]:
    if not dist.is_available() or not dist.is_initialized():
        return 0, 1
    return dist.get_rank(group), dist.get_world_size(group)


def shard_window(n_items: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous [lo, hi) window of n_items for rank (sizes differ by <= 1)."""
    base, extra = divmod(int(n_items), int(world))
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def mix64(keys) -> np.ndarray:
    """The device's 64-bit finaliser (csrc/vhash.cu mix64) on uint64 keys."""
    k = np.asarray(keys).astype(np.uint64)
    with np.errstate(over="ignore"):
        k = k ^ (k >> np.uint64(33))
        k = k * np.uint64(_M1)
        k = k ^ (k >> np.uint64(33))
        k = k * np.uint64(_M2)
        k = k ^ (k >> np.uint64(33))
    return k


def owner_of(keys, world: int) -> np.ndarray:
    """Owner rank of packed voxel keys: mix64(key) mod world (device rule)."""
    return (mix64(keys) % np.uint64(world)).astype(np.int64)


def _host_staged(group, dev) -> bool:
    """gloo moves CPU tensors only: CUDA payloads are staged through host
    memory (validation runs with several ranks per GPU); NCCL moves them
    directly over NVLink."""
    return dev.type == "cuda" and dist.get_backend(group) == "gloo"


def gather_ragged(t: torch.Tensor, group=None) -> list[torch.Tensor]:
    """All-gather tensors whose first dimension differs per rank."""
    rank, world = _world(group)
    if world == 1:
        return [t]
    if _host_staged(group, t.device):
        return [x.to(t.device) for x in gather_ragged(t.cpu(), group)]
    n = torch.tensor([t.shape[0]], dtype=torch.int64, device=t.device)
    sizes = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(sizes, n, group=group)
    sizes = [int(s.item()) for s in sizes]
    m = max(max(sizes), 1)
    pad = torch.zeros((m,) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
    pad[: t.shape[0]] = t
    bufs = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(bufs, pad, group=group)
    return [b[:s] for b, s in zip(bufs, sizes)]


def exchange_partials(keys: torch.Tensor, sums4: torch.Tensor, counts: torch.Tensor,
                      rank_counts: Sequence[int], group=None):
    """One all-to-all of owner-bucketed partials.

    keys (n,) int64, sums4 (n, 4) float32, counts (n,) int32, laid out as
    contiguous per-owner buckets of sizes rank_counts (the layout
    ec3r_vhash_extract_partials writes).  Returns the partials this rank
    owns, received from every rank (rank order)."""
    rank, world = _world(group)
    send = [int(c) for c in rank_counts]
    if world == 1:
        return keys[: send[0]], sums4[: send[0]], counts[: send[0]]
    dev = keys.device
    if _host_staged(group, dev):
        k, s_, c = exchange_partials(keys.cpu(), sums4.cpu(), counts.cpu(), rank_counts, group)
        return k.to(dev), s_.to(dev), c.to(dev)
    sc = torch.tensor(send, dtype=torch.int64, device=dev)
    rc = torch.empty_like(sc)
    dist.all_to_all_single(rc, sc, group=group)
    recv = [int(x) for x in rc.tolist()]
    n_in = sum(recv)
    n_out = sum(send)
    # one packed payload per row: key (2 x int32 words), 4 float sums, count
    def pack(k, s, c):
        return torch.cat([k.view(torch.int32).reshape(-1, 2), s.view(torch.int32).reshape(-1, 4),
                          c.reshape(-1, 1).to(torch.int32)], dim=1)
    payload = pack(keys[:n_out], sums4[:n_out], counts[:n_out])
    out = torch.empty((n_in, 7), dtype=torch.int32, device=dev)
    dist.all_to_all_single(out, payload, output_split_sizes=recv, input_split_sizes=send, group=group)
    k = out[:, 0:2].contiguous().view(torch.int64).reshape(-1)
    s = out[:, 2:6].contiguous().view(torch.float32)
    c = out[:, 6].contiguous()
    return k, s, c


class MapExchange:
    """Owner-partitioned global voxel map from per-rank local maps, with no
    host round trip in the step: the partials of a rank's local VoxelMap are
    bucketed by owner on the device into fixed slabs of `cap` rows
    (ec3r_vhash_extract_partials_fixed), so the bucket counts and the payload
    each move in one equal-split all-to-all (counts stay on the device), and
    the owner merges the received slabs with their device counts
    (ec3r_vhash_merge_partials_slabs) before its sorted emit.  Overflow (a
    bucket larger than `cap`, or the owned map's capacity) is flagged on the
    device: run(sync=True) checks it and re-runs with larger buffers;
    run(sync=False) returns the unsliced outputs plus the device count and
    leaves the check to verify().  Buffers persist across calls."""

    def __init__(self, cell: float, group=None, cap: Optional[int] = None):
        self.cell = float(cell)
        self.group = group
        self.rank, self.world = _world(group)
        self.cap = int(cap) if cap else 0
        self.owned = None
        self._bufs = None
        self.out = None
        self.flags = None  # device int64[2]: partition overflow, owned-map overflow (accumulated)
        self._stats = None
        self._slab = None

    def _alloc(self, cap: int):
        W = self.world
        dev = torch.device("cuda", torch.cuda.current_device())
        n = W * cap
        self._bufs = dict(
            keys=torch.empty(n, dtype=torch.int64, device=dev),
            sums4=torch.empty((n, 4), dtype=torch.float32, device=dev),
            cnt=torch.empty(n, dtype=torch.int32, device=dev),
            send_counts=torch.zeros(W, dtype=torch.int64, device=dev),
            recv_counts=torch.zeros(W, dtype=torch.int64, device=dev),
            payload=torch.empty((n, 7), dtype=torch.int32, device=dev),
            recv=torch.empty((n, 7), dtype=torch.int32, device=dev),
            ovf=torch.zeros(1, dtype=torch.int64, device=dev))
        from .mapping import VoxelMap
        self.owned = VoxelMap(self.cell, capacity=max(n, 1 << 16))
        self.out = (torch.empty(max(n, 1), dtype=torch.int64, device=dev),
                    torch.empty((max(n, 1), 3), dtype=torch.float32, device=dev),
                    torch.empty(max(n, 1), dtype=torch.float32, device=dev),
                    torch.empty(max(n, 1), dtype=torch.int32, device=dev))
        self.flags = torch.zeros(2, dtype=torch.int64, device=dev)
        self._stats = torch.zeros(5, dtype=torch.int64, device=dev)
        self.cap = cap

    def _all_to_all(self, out: torch.Tensor, inp: torch.Tensor):
        if _host_staged(self.group, inp.device):
            o = torch.empty_like(out, device="cpu")
            dist.all_to_all_single(o, inp.cpu(), group=self.group)
            out.copy_(o)
        else:
            dist.all_to_all_single(out, inp, group=self.group)

    def run(self, local, n_local: int, stream=None, sync: bool = True):
        """local: this rank's fused VoxelMap holding ~n_local voxels.
        sync=True: returns (keys, centroid, wsum, count) sliced to this rank's
        partition, re-running with larger slabs on overflow (all ranks agree
        through one all-reduce of the flags).  sync=False: returns the full
        output buffers and the device int64[1] count; no host round trip."""
        if self._bufs is None:
            cap = self.cap or max(1024, (2 * int(n_local)) // max(self.world, 1) + 1024)
            if self.world > 1:  # equal splits: every rank uses the largest slab any rank needs
                t = torch.tensor([cap], dtype=torch.int64, device=_coll_dev(self.group))
                dist.all_reduce(t, op=dist.ReduceOp.MAX, group=self.group)
                cap = int(t.item())
            self._alloc(cap)
        while True:
            if sync:
                self.flags.zero_()
            res = self._step(local, stream)
            if not sync:
                return res
            f = self.flags.clone()
            if self.world > 1:
                if _host_staged(self.group, f.device):
                    fc = f.cpu()
                    dist.all_reduce(fc, op=dist.ReduceOp.MAX, group=self.group)
                    f = fc
                else:
                    dist.all_reduce(f, op=dist.ReduceOp.MAX, group=self.group)
            if int(f.max().item()) == 0:
                n = int(res[4].item())
                return tuple(x[:n] for x in res[:4])
            self._alloc(2 * self.cap)

    def _step(self, local, stream):
        from . import _lib

        L = _lib.lib()
        b, W, cap = self._bufs, self.world, self.cap
        wsb = L.ec3r_vhash_extract_workspace(local.handle) + 2 * 256 * max(W, 4) + 4096
        ws = _lib.workspace(wsb, b["keys"].device, "partials")
        _lib.check(L.ec3r_vhash_extract_partials_fixed(local.handle, W, cap, _lib.ptr(b["keys"]), _lib.ptr(b["sums4"]),
                                                       _lib.ptr(b["cnt"]), _lib.ptr(b["send_counts"]),
                                                       _lib.ptr(b["ovf"]), _lib.ptr(ws), ws.numel(),
                                                       _lib.stream_ptr(stream)), "ec3r_vhash_extract_partials_fixed")
        self.flags[0:1].add_(b["ovf"])
        p = b["payload"]
        p[:, 0:2].copy_(b["keys"].view(torch.int32).view(-1, 2))
        p[:, 2:6].copy_(b["sums4"].view(torch.int32))
        p[:, 6].copy_(b["cnt"])
        if W > 1:
            self._all_to_all(b["recv_counts"], b["send_counts"])
            self._all_to_all(b["recv"], p)
            r, counts = b["recv"], b["recv_counts"]
        else:
            r, counts = p, b["send_counts"]
        rk = r[:, 0:2].contiguous().view(torch.int64).view(-1)
        rs = r[:, 2:6].contiguous().view(torch.float32)
        rc = r[:, 6].contiguous()
        self.owned.clear(stream)
        _lib.check(L.ec3r_vhash_merge_partials_slabs(self.owned.handle, _lib.ptr(rk), _lib.ptr(rs), _lib.ptr(rc), W,
                                                     cap, _lib.ptr(counts), _lib.stream_ptr(stream)),
                   "ec3r_vhash_merge_partials_slabs")
        res = self.owned.extract(sort=True, stream=stream, out=self.out, sync=False)
        self.owned.stats_device(self._stats, stream)
        self.flags[1:2].add_(self._stats[2:3])
        return res

    def retune(self, slack: float = 1.1):
        """Shrink (or grow) the slabs to `slack` x the largest bucket any rank
        sent in the last run (one all-reduce; call outside timed loops).  The
        equal-split all-to-all moves world x cap rows per rank, so the slab
        size is the traffic: hash-partitioned buckets are balanced, and the
        first sizing (2 x n_local / world) is twice what they need."""
        b = self._bufs
        if b is None:
            return self.cap
        m = b["send_counts"].max().reshape(1).clone()
        if self.world > 1:
            if _host_staged(self.group, m.device):
                mc = m.cpu()
                dist.all_reduce(mc, op=dist.ReduceOp.MAX, group=self.group)
                m = mc
            else:
                dist.all_reduce(m, op=dist.ReduceOp.MAX, group=self.group)
        f = self.flags.clone()
        if self.world > 1:
            if _host_staged(self.group, f.device):
                fc = f.cpu()
                dist.all_reduce(fc, op=dist.ReduceOp.MAX, group=self.group)
                f = fc
            else:
                dist.all_reduce(f, op=dist.ReduceOp.MAX, group=self.group)
        if int(f.max().item()):  # the last run overflowed: its counts are clipped
            cap = 2 * self.cap
        else:
            cap = max(1024, int(math.ceil(slack * int(m.item()))) + 64)
        if cap != self.cap:
            self._alloc(cap)
        return cap

    def verify(self):
        """Host check of the overflow flags accumulated by run(sync=False)."""
        f = self.flags.tolist()
        if f[0] or f[1]:
            raise RuntimeError(f"MapExchange overflow: {f[0]} partial rows past a slab of {self.cap}, "
                               f"{f[1]} rows past the owned map; re-run with a larger cap")


def fuse_global(pool, slots: torch.Tensor, cell: float, group=None, capacity: Optional[int] = None):
    """Global voxel map over all ranks' frames: local fusion, owner-bucketed
    partials, one all-to-all, owner-side merge.  Returns this rank's owned
    partition (keys sorted ascending, centroid, wsum, count)."""
    from .mapping import fuse_slots

    local, out, _ = fuse_slots(pool, slots, cell, expected_voxels=capacity)
    if _world(group)[1] == 1:
        return out
    return MapExchange(cell, group).run(local, int(out[0].shape[0]))


def retrieval_sharded(db, stride: int, exclusion: int, tau_g: float, tau_l: float, group=None):
    """Sharded K6: rank r scores the coarse rows of its window; the lists
    concatenated in rank order are the single-GPU lists (reference emission
    order).  Returns the six numpy arrays of loops.retrieval_device."""
    rank, world = _world(group)
    kc = (db.n + stride - 1) // stride
    lo, hi = shard_window(kc, world, rank)
    parts = db.score(stride, exclusion, tau_g, tau_l, lo, hi)
    if world == 1:
        return parts
    dev = db.vec.device
    merged = []
    for a in parts:
        t = torch.as_tensor(np.ascontiguousarray(a), device=dev)
        merged.append(torch.cat(gather_ragged(t, group)).cpu().numpy())
    return tuple(merged)


# -- align windows with a shared-frame halo (SURVEY.md §8(e), row (a)+(b)) --
#
# Rank r owns a contiguous window of submaps.  Its first submap shares a
# keyframe with the last submap of rank r-1 (KeyframeBuffer flush order,
# loops.py:89-111), so registering it needs the predecessor's copy of that
# frame: a halo of one 392x518 depth + confidence plane (1.6 MB) and its
# local pose.  Each rank registers [halo stub] + window with the stub fixed
# at identity (mapping.py:190-211 semantics), which gives every submap's
# pose relative to the predecessor's last submap; one all-gather of the
# windows' last poses (8 f64 per rank) and a prefix composition in rank
# order turn those into global poses.  Edge measurements never depend on
# global poses, so the result equals single-process registration up to the
# association order of the Sim(3) compositions.

HALO_MAX = 16  # keyframes one submap may share with its predecessor


def _peer(group, r: int) -> int:
    return r if group is None else dist.get_global_rank(group, r)


def shift(send: Sequence[torch.Tensor], recv: Sequence[torch.Tensor], step: int = 1, group=None) -> None:
    """Grouped P2P: rank r sends `send` to rank r+step and receives `recv`
    (preallocated, same shapes as the sender's) from rank r-step; ranks at
    the ends skip the side that does not exist."""
    rank, world = _world(group)
    if world == 1:
        return
    ops = []
    dst, src = rank + step, rank - step
    if 0 <= dst < world:
        ops += [dist.P2POp(dist.isend, t.contiguous(), _peer(group, dst), group) for t in send]
    if 0 <= src < world:
        ops += [dist.P2POp(dist.irecv, t, _peer(group, src), group) for t in recv]
    if ops:
        for w in dist.batch_isend_irecv(ops):
            w.wait()


def window_halo(mapping, window: Sequence, group=None):
    """Fetch the predecessor's halo and add it to `mapping` as a stub submap.

    Two point-to-point rounds: rank r sends the keyframe ids of its first
    submap to rank r-1; rank r-1 answers with the frames of its last submap
    holding those keyframes (ids, depth, confidence, local pose).  Returns the
    stub (None on rank 0, or when nothing is shared)."""
    rank, world = _world(group)
    if world == 1:
        return None
    pool = mapping.pool
    dev = pool.device
    tdev = torch.device("cpu") if _host_staged(group, dev) else dev
    H, W = pool.H, pool.W
    i64 = dict(dtype=torch.int64, device=tdev)
    # round 1 (backwards): requested keyframe ids, -1 padded
    req = torch.full((HALO_MAX,), -1, **i64)
    if window:
        ids = list(window[0].keyframe_ids)[:HALO_MAX]
        req[: len(ids)] = torch.tensor(ids, dtype=torch.int64)
    want = torch.full((HALO_MAX,), -1, **i64)
    shift([req], [want], step=-1, group=group)
    # round 2 (forwards): header (count, submap id, ids) then the frames
    send = []
    if rank + 1 < world:
        wanted = {int(x) for x in want.tolist() if x >= 0}
        last = window[-1]
        pick = [k for k, f in enumerate(last.keyframe_ids) if f in wanted]
        hdr = torch.full((2 + HALO_MAX,), -1, **i64)
        hdr[0] = len(pick)
        hdr[1] = int(last.id)
        hdr[2: 2 + len(pick)] = torch.tensor([last.keyframe_ids[k] for k in pick], dtype=torch.int64)
        sl = torch.as_tensor(np.asarray(last.slots, np.int64)[pick], device=dev)
        send = [hdr, pool.depth.index_select(0, sl).to(tdev), pool.conf.index_select(0, sl).to(tdev),
                pool.poses.index_select(0, sl).to(tdev)]
        n_send = len(pick)
    hdr_in = torch.full((2 + HALO_MAX,), -1, **i64)
    shift(send[:1], [hdr_in] if rank > 0 else [], step=1, group=group)
    n_in = int(hdr_in[0]) if rank > 0 else 0
    recv = []
    if rank > 0 and n_in > 0:
        recv = [torch.empty((n_in, H, W), dtype=pool.depth.dtype, device=tdev),
                torch.empty((n_in, H, W), dtype=pool.conf.dtype, device=tdev),
                torch.empty((n_in, 8), dtype=torch.float64, device=tdev)]
    shift(send[1:] if rank + 1 < world and n_send > 0 else [], recv, step=1, group=group)
    if rank == 0 or n_in == 0:
        return None
    ids = [int(x) for x in hdr_in[2: 2 + n_in].tolist()]
    stub = mapping.add_submap(ids, recv[0].to(dev), recv[1].to(dev), list(recv[2].cpu().numpy()))
    mapping._next_id -= 1  # the stub takes no id of this rank's sequence
    stub.id = -(1 << 30)
    stub.remote_id = int(hdr_in[1])  # the predecessor's submap (global id): edges name it
    return stub


def prefix_offsets(window_last: Sequence) -> list:
    """O_0 = identity, O_r = O_{r-1} o W_{r-1}: the global pose of each
    window's reference frame from the windows' last-submap poses W_r (each
    expressed in its own window's frame).  Sim(3) 8-vectors."""
    from .types import Sim3Transform, sim3_to_vec, vec_to_sim3

    out = [sim3_to_vec(Sim3Transform.identity())]
    for w in list(window_last)[:-1]:
        out.append(sim3_to_vec(vec_to_sim3(out[-1]).compose(vec_to_sim3(np.asarray(w, np.float64)))))
    return [np.asarray(o, np.float64) for o in out]


def window_offset(last_local, group=None, device=None) -> np.ndarray:
    """All-gather every window's last-submap pose (8 f64 per rank) and return
    this rank's prefix offset (prefix_offsets)."""
    rank, world = _world(group)
    v = np.asarray(last_local, np.float64).reshape(8)
    if world == 1:
        return prefix_offsets([v])[0]
    dev = torch.device("cpu") if device is None else torch.device(device)
    if _host_staged(group, dev):
        dev = torch.device("cpu")
    t = torch.as_tensor(v, device=dev)
    bufs = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(bufs, t, group=group)
    return prefix_offsets([b.cpu().numpy() for b in bufs])[rank]


def register_window(mapping, window: Sequence, group=None):
    """Register this rank's window of submaps into global poses.

    `mapping` holds only this rank's submaps (window, in order).  The halo
    stub is registered first (identity), used as the first submap's partner
    and then forgotten, so fusion never sees the predecessor's frames twice.
    Returns the window offset (Sim3Transform)."""
    from .types import sim3_to_vec, vec_to_sim3

    stub = window_halo(mapping, window, group)
    n0 = len(mapping.edges)
    mapping.register_chain(([stub] if stub is not None else []) + list(window))
    if stub is not None:  # the halo edge names the predecessor's submap, not the stub
        mapping.edges[n0:] = [(stub.remote_id if i == stub.id else i, j, tr, info)
                              for i, j, tr, info in mapping.edges[n0:]]
    off = vec_to_sim3(window_offset(sim3_to_vec(window[-1].global_pose), group, mapping.pool.device))
    if stub is not None:
        mapping.forget(stub)
    for sm in window:
        sm.global_pose = off.compose(sm.global_pose)
        mapping._commit(sm)
    return off


def halo_handshake(first_ids: Sequence[int], last_ids: Sequence[int], group=None):
    """Agree on the halo once, before the pools are filled.  Rank r sends the
    keyframe ids of its first submap back to rank r-1, which answers with the
    ones its last submap holds.  Returns (send_pos, recv_ids): positions in
    this rank's last submap to send forward each step, and the keyframe ids
    of the frames arriving from the predecessor (empty on rank 0)."""
    rank, world = _world(group)
    if world == 1:
        return [], []
    dev = torch.device("cpu")
    if dist.get_backend(group) == "nccl":
        dev = torch.device("cuda", torch.cuda.current_device())
    req = torch.full((HALO_MAX,), -1, dtype=torch.int64, device=dev)
    ids = list(first_ids)[:HALO_MAX]
    if ids:
        req[: len(ids)] = torch.tensor(ids, dtype=torch.int64)
    want = torch.full_like(req, -1)
    shift([req], [want], step=-1, group=group)
    send_pos = []
    hdr = torch.full((HALO_MAX,), -1, dtype=torch.int64, device=dev)
    if rank + 1 < world:
        wanted = {int(x) for x in want.tolist() if x >= 0}
        send_pos = [k for k, f in enumerate(last_ids) if int(f) in wanted][:HALO_MAX]
        if send_pos:
            hdr[: len(send_pos)] = torch.tensor([int(last_ids[k]) for k in send_pos], dtype=torch.int64)
    got = torch.full_like(hdr, -1)
    shift([hdr], [got], step=1, group=group)
    recv_ids = [int(x) for x in got.tolist() if x >= 0] if rank > 0 else []
    return send_pos, recv_ids


class WindowChain:
    """Device-resident sharded registration chain (ChainPlan over
    [halo stub] + window) with the per-step exchange steps of SURVEY §8(e):

    1. grouped isend / irecv of the halo frames (depth, confidence, local
       pose) from rank r-1's last submap into this rank's stub slots;
    2. registration of every edge + device pose chain (ChainPlan.run), the
       stub fixed at identity;
    3. all-gather of each window's last-submap pose (8 f64 per rank) and
       ec3r_apply_window_offset, which left-composes the prefix offset into
       the submap and slot globals.

    No host synchronisation; with NCCL all transfers stay on the device."""

    def __init__(self, dm, stub, window: Sequence, send_pos: Sequence[int], group=None):
        from .mapping import ChainPlan

        self.rank, self.world = _world(group)
        self.group, self.dm, self.stub, self.window = group, dm, stub, list(window)
        self.plan = ChainPlan(([stub] if stub is not None else []) + self.window, device=dm.pool.device)
        pool = dm.pool
        self.send_slots = [int(self.window[-1].slots[k]) for k in send_pos] if self.window else []
        self.staged = self.world > 1 and _host_staged(group, pool.device)
        self.last = torch.zeros(8, dtype=torch.float64, device=pool.device)
        self.gathered = torch.zeros((max(self.world, 1), 8), dtype=torch.float64, device=pool.device)
        self.offset = torch.zeros(8, dtype=torch.float64, device=pool.device)
        self.n_slots = sum(len(sm.slots) for sm in self.plan.sms)

    def _halo(self):
        pool = self.dm.pool
        send, recv = [], []
        for s in self.send_slots:
            send += [pool.depth[s:s + 1], pool.conf[s:s + 1], pool.poses[s:s + 1]]
        if self.stub is not None:
            s0, s1 = int(self.stub.slots[0]), int(self.stub.slots[-1]) + 1
            recv = [t[s:s + 1] for s in range(s0, s1) for t in (pool.depth, pool.conf, pool.poses)]
        if self.staged:
            hs = [t.cpu() for t in send]
            hr = [torch.empty_like(t, device="cpu") for t in recv]
            shift(hs, hr, step=1, group=self.group)
            for d, h in zip(recv, hr):
                d.copy_(h)
        else:
            shift(send, recv, step=1, group=self.group)

    def run(self, config=None, stream=None):
        from . import _lib
        from .mapping import MappingConfig

        if self.world > 1:
            self._halo()
        out = self.plan.run(self.dm.pool, config or MappingConfig(), stream=stream)
        sub_globals = out[5]
        if self.world > 1:
            self.last.copy_(sub_globals[-1])
            if self.staged:
                bufs = [torch.empty(8, dtype=torch.float64) for _ in range(self.world)]
                dist.all_gather(bufs, self.last.cpu(), group=self.group)
                self.gathered.copy_(torch.stack(bufs))
            else:
                dist.all_gather_into_tensor(self.gathered, self.last, group=self.group)
            pool = self.dm.pool
            slot_g = pool.globals[self.plan.slot0:]
            n_slots = self.n_slots
            _lib.check(_lib.lib().ec3r_apply_window_offset(_lib.ptr(self.gathered), self.world, self.rank,
                                                           _lib.ptr(sub_globals), int(sub_globals.shape[0]),
                                                           _lib.ptr(slot_g), n_slots, _lib.ptr(self.offset),
                                                           _lib.stream_ptr(stream)), "ec3r_apply_window_offset")
        return out


# -- loop edges across shards and the pose-graph data path ----
#
# Submap ids are global: every rank numbers its window from the window's
# first global index (DenseMapping._next_id), so an edge (i, j) means the same
# submaps on every rank.  A loop submap (mapping.py:282-318) is registered
# against every submap sharing one of its keyframes -- those may live on any
# shard.  The owner of the loop submap requests the shared frames (depth,
# confidence, local pose, plus the partner's global pose) from their owners
# in one ragged all-to-all, adds them as stub submaps, registers every edge
# in one launch, chains the loop submap off its strongest partner and drops
# the stubs again.  Pose-graph optimisation stays in the reference's host
# code (posegraph.py:176): the per-edge results (i, j, s, q, t, count, rms)
# and every submap's global pose are gathered to the PGO rank, which runs the
# caller's optimiser and broadcasts the optimised poses (8 f64 per submap);
# each rank re-commits its own submaps (slot globals on the device).

def _coll_dev(group=None) -> torch.device:
    """Device of small host-side collectives: NCCL moves CUDA tensors only."""
    if dist.is_available() and dist.is_initialized() and dist.get_backend(group) == "nccl":
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device("cpu")


class SubmapDirectory:
    """Replicated directory of every rank's committed submaps: owner rank and
    keyframe ids (one ragged all-gather of (sid, keyframe) rows; collective)."""

    def __init__(self, mapping, group=None):
        self.group = group
        self.rank, self.world = _world(group)
        rows = [(sid, kf, self.rank) for sid, sm in mapping.submaps.items() for kf in sm.keyframe_ids]
        t = torch.as_tensor(np.asarray(rows, np.int64).reshape(-1, 3), device=_coll_dev(group))
        parts = [x.cpu() for x in gather_ragged(t, group)] if self.world > 1 else [t]
        self.owner: dict = {}
        self.kf_subs: dict = {}
        self.sub_kfs: dict = {}
        for p in parts:
            for sid, kf, r in p.tolist():
                self.owner[sid] = r
                self.kf_subs.setdefault(kf, []).append(sid)
                self.sub_kfs.setdefault(sid, []).append(kf)

    def partners(self, keyframe_ids, exclude=None) -> list:
        """Submaps sharing any of keyframe_ids (mapping.py:164-169 order:
        keyframes in order, then the submaps holding each)."""
        out: dict = {}
        for kf in keyframe_ids:
            for sid in self.kf_subs.get(int(kf), ()):
                if sid != exclude:
                    out[sid] = None
        return list(out)


def _a2a_ragged(send: list, dtype, width: int, dev, group) -> list:
    """Ragged all-to-all of per-destination row blocks (each (n_r, width)
    of `dtype`); returns the blocks received from every rank.  Sizes travel
    first (one host read: this path is per loop closure, not per frame)."""
    rank, world = _world(group)
    sizes = torch.tensor([int(b.shape[0]) for b in send], dtype=torch.int64)
    rs = torch.empty_like(sizes)
    staged = dev.type == "cpu" or dist.get_backend(group) == "gloo"
    sdev = torch.device("cpu") if staged else dev
    if staged:
        dist.all_to_all_single(rs, sizes, group=group)
    else:
        s_d, r_d = sizes.to(dev), torch.empty(world, dtype=torch.int64, device=dev)
        dist.all_to_all_single(r_d, s_d, group=group)
        rs = r_d.cpu()
    recv_sizes = [int(x) for x in rs.tolist()]
    flat = torch.cat([b.reshape(-1, width).to(device=sdev, dtype=dtype) for b in send]) if send else \
        torch.empty((0, width), dtype=dtype, device=sdev)
    out = torch.empty((sum(recv_sizes), width), dtype=dtype, device=sdev)
    dist.all_to_all_single(out, flat.contiguous(), output_split_sizes=recv_sizes,
                           input_split_sizes=[int(b.shape[0]) for b in send], group=group)
    res, o = [], 0
    for n in recv_sizes:
        res.append(out[o:o + n].to(dev))
        o += n
    return res


def fetch_frames(mapping, requests, directory: SubmapDirectory, group=None) -> dict:
    """Collective: every rank passes the (submap id, keyframe id) frames it
    needs (possibly none); owners answer with that submap's copy of the frame.
    Returns {(sid, kf): (depth (H,W) f32, conf (H,W) f32, local pose 8 f64,
    submap global pose 8 f64)} on the pool's device."""
    rank, world = _world(group)
    pool = mapping.pool
    dev = pool.device
    H, W = pool.H, pool.W
    per = [[] for _ in range(world)]
    for sid, kf in requests:
        per[directory.owner[int(sid)]].append((int(sid), int(kf)))
    if world == 1:
        incoming = [torch.as_tensor(np.asarray(per[0], np.int64).reshape(-1, 2))]
    else:
        incoming = _a2a_ragged([torch.as_tensor(np.asarray(p, np.int64).reshape(-1, 2)) for p in per],
                               torch.int64, 2, _coll_dev(group), group)
    from .types import sim3_to_vec

    planes, poses = [], []
    for blk in incoming:
        rows = blk.cpu().tolist()
        if not rows:
            planes.append(torch.empty((0, 2 * H * W), dtype=torch.float32, device=dev))
            poses.append(torch.empty((0, 16), dtype=torch.float64, device=dev))
            continue
        sl = []
        gl = []
        for sid, kf in rows:
            sm = mapping.submaps[sid]
            sl.append(int(sm.slots[list(sm.keyframe_ids).index(kf)]))
            gl.append(sim3_to_vec(sm.global_pose))
        idx = torch.as_tensor(np.asarray(sl, np.int64), device=dev)
        planes.append(torch.cat([pool.depth.index_select(0, idx).reshape(len(sl), -1),
                                 pool.conf.index_select(0, idx).reshape(len(sl), -1)], dim=1))
        poses.append(torch.cat([pool.poses.index_select(0, idx),
                                torch.as_tensor(np.asarray(gl, np.float64), device=dev)], dim=1))
    if world == 1:
        got_planes, got_poses = planes, poses
    else:
        got_planes = _a2a_ragged(planes, torch.float32, 2 * H * W, dev, group)
        got_poses = _a2a_ragged(poses, torch.float64, 16, dev, group)
    out = {}
    for r in range(world):
        for k, (sid, kf) in enumerate(per[r]):
            pl = got_planes[r][k]
            ps = got_poses[r][k]
            out[(sid, kf)] = (pl[: H * W].reshape(H, W), pl[H * W:].reshape(H, W), ps[:8].cpu().numpy(),
                              ps[8:].cpu().numpy())
    return out


def register_loop_sharded(mapping, loop_sm, directory: SubmapDirectory, group=None):
    """Collective (every rank calls; loop_sm is None on ranks without a loop
    submap this step).  Registers loop_sm against every submap, on any shard,
    sharing one of its keyframes (mapping.py:282-318 with _registration_edges
    :162-188), sets its global pose from the strongest partner and commits it.
    Returns the edges [(partner id, loop id, T, info, count, rms)] (empty when
    there is no loop submap, or NoSharedKeyframes: the graph stays untouched,
    mapping.py:309-311)."""
    from .types import NoSharedKeyframes, vec_to_sim3

    rank, world = _world(group)
    requests, local_p, remote_p = [], [], {}
    if loop_sm is not None:
        for sid in directory.partners(loop_sm.keyframe_ids, exclude=loop_sm.id):
            if directory.owner[sid] == rank and sid in mapping.submaps:
                local_p.append(sid)
            else:
                shared = [kf for kf in directory.sub_kfs[sid] if kf in loop_sm.keyframe_ids]
                remote_p[sid] = shared
                requests += [(sid, kf) for kf in shared]
    frames = fetch_frames(mapping, requests, directory, group)
    if loop_sm is None:
        return []
    stubs, order = {}, []
    for sid in directory.partners(loop_sm.keyframe_ids, exclude=loop_sm.id):
        if sid in remote_p:
            kfs = remote_p[sid]
            d = torch.stack([frames[(sid, kf)][0] for kf in kfs])
            c = torch.stack([frames[(sid, kf)][1] for kf in kfs])
            p8 = [frames[(sid, kf)][2] for kf in kfs]
            st = mapping.add_submap(kfs, d, c, p8)
            mapping._next_id -= 1  # stubs take no id of this rank's sequence
            st.id = -1 - len(stubs)
            st.global_pose = vec_to_sim3(frames[(sid, kfs[0])][3])
            mapping.submaps[st.id] = st  # a partner for this registration only
            stubs[st.id] = sid
            order.append(st.id)
        else:
            order.append(sid)
    try:
        edges = mapping.registration_edges(loop_sm, partner_ids=order)
    except NoSharedKeyframes:
        edges = []
    best = max(edges, key=lambda e: e[3]) if edges else None
    if best is not None:
        loop_sm.global_pose = mapping.submaps[best[0]].global_pose.compose(best[1])
    for st_id in stubs:
        mapping.submaps.pop(st_id, None)
    if best is None:
        return []
    mapping._commit(loop_sm)
    out = []
    for sid, tr, info, count, rms in edges:
        gid = stubs.get(sid, sid)
        mapping.edges.append((gid, loop_sm.id, tr, info))
        out.append((gid, loop_sm.id, tr, info, count, rms))
    return out


EDGE_COLS = 12  # i, j, s, qw, qx, qy, qz, tx, ty, tz, information scale, (pad)


def edge_rows(edges) -> np.ndarray:
    """(i, j, T, info, ...) tuples -> (n, EDGE_COLS) float64 rows."""
    from .types import sim3_to_vec

    rows = np.zeros((len(edges), EDGE_COLS), np.float64)
    for k, e in enumerate(edges):
        i, j, tr, info = e[:4]
        rows[k, 0], rows[k, 1] = i, j
        rows[k, 2:10] = sim3_to_vec(tr)
        rows[k, 10] = float(np.asarray(info)[0, 0]) if np.ndim(info) == 2 else float(info)
    return rows


def gather_graph(mapping, edges, group=None, root: int = 0):
    """Collective: (node poses {sid: 8 f64}, edge rows (n, EDGE_COLS)) of all
    ranks, on `root` (None elsewhere)."""
    from .types import sim3_to_vec

    rank, world = _world(group)
    nodes = np.asarray([[sid, *sim3_to_vec(sm.global_pose)] for sid, sm in mapping.submaps.items()],
                       np.float64).reshape(-1, 9)
    er = edge_rows(edges)
    if world == 1:
        return {int(r[0]): r[1:] for r in nodes}, er
    cd = _coll_dev(group)
    n_parts = [x.cpu() for x in gather_ragged(torch.as_tensor(nodes, device=cd), group)]
    e_parts = [x.cpu() for x in gather_ragged(torch.as_tensor(er, device=cd), group)]
    if rank != root:
        return None, None
    allnodes = {int(r[0]): r[1:].copy() for p in n_parts for r in p.numpy()}
    return allnodes, np.concatenate([p.numpy() for p in e_parts]) if e_parts else er[:0]


def broadcast_poses(poses, ids, group=None, root: int = 0) -> dict:
    """Collective: the root's {sid: 8 f64} for the listed ids to every rank."""
    rank, world = _world(group)
    t = torch.zeros((len(ids), 8), dtype=torch.float64)
    if rank == root and ids:
        t[:] = torch.as_tensor(np.stack([np.asarray(poses[i], np.float64) for i in ids]))
    if world > 1:
        td = t.to(_coll_dev(group))
        dist.broadcast(td, src=_peer(group, root), group=group)
        t = td.cpu()
    return {int(i): t[k].numpy() for k, i in enumerate(ids)}


def optimize_sharded(mapping, edges, optimize_fn, group=None, root: int = 0) -> dict:
    """Collective pose-graph step: gather every node and edge to `root`, run
    optimize_fn(nodes {sid: 8 f64}, edge_rows) -> {sid: 8 f64} there (the
    reference's host PGO, posegraph.py:176), broadcast the result and
    re-commit this rank's submaps (their pool slot globals on the device).
    Returns the optimised poses of all submaps."""
    from .types import vec_to_sim3

    rank, world = _world(group)
    nodes, rows = gather_graph(mapping, edges, group, root)
    ids = None
    if rank == root:
        new = optimize_fn(nodes, rows)
        ids = sorted(new)
    cd = _coll_dev(group)
    idt = torch.as_tensor(np.asarray(ids if ids is not None else [], np.int64), device=cd)
    if world > 1:
        n = torch.tensor([idt.numel()], dtype=torch.int64, device=cd)
        dist.broadcast(n, src=_peer(group, root), group=group)
        if rank != root:
            idt = torch.zeros(int(n.item()), dtype=torch.int64, device=cd)
        dist.broadcast(idt, src=_peer(group, root), group=group)
    ids = [int(x) for x in idt.cpu().tolist()]
    out = broadcast_poses(new if rank == root else None, ids, group, root)
    for sid, v in out.items():
        sm = mapping.submaps.get(sid)
        if sm is not None:
            sm.global_pose = vec_to_sim3(v)
            mapping._commit(sm)
    return out


def _reference_posegraph():
    """submap_slam.posegraph / liegroups: importable as installed, or from
    EC3R_REFERENCE_SRC, or from the offline install under baseline/_ref."""
    import importlib
    import os
    import sys

    try:
        return importlib.import_module("submap_slam.posegraph"), importlib.import_module("submap_slam.liegroups")
    except ImportError:
        root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
        for p in (os.environ.get("EC3R_REFERENCE_SRC"), os.path.join(root, "baseline", "_ref")):
            if p and os.path.isdir(p) and p not in sys.path:
                sys.path.append(p)
        return importlib.import_module("submap_slam.posegraph"), importlib.import_module("submap_slam.liegroups")


def reference_pgo(lm_config=None):
    """optimize_fn running the reference's own PoseGraph (posegraph.py:93-255,
    host code by design) on reference Sim3Transform values built from the
    8-vectors: the first node (smallest id) is fixed, as the reference fixes
    its first submap (mapping.py:194-197).  Raises ImportError without the
    reference."""
    pg, lg = _reference_posegraph()

    def to_ref(v):
        v = np.asarray(v, np.float64)
        return lg.Sim3Transform(float(v[0]), lg.Rotation3(v[1:5]), v[5:8])

    def fn(nodes, rows):
        g = pg.PoseGraph()
        first = min(nodes)
        for sid in sorted(nodes):
            g.add_node(sid, to_ref(nodes[sid]), fixed=(sid == first))
        for r in rows:
            g.add_edge(int(r[0]), int(r[1]), to_ref(r[2:10]), np.eye(7) * float(r[10]))
        g.optimize(lm_config or pg.LmConfig())
        return {sid: np.concatenate([[float(n.pose.scale)], np.asarray(n.pose.rotation.q, float),
                                     np.asarray(n.pose.translation, float)]) for sid, n in g.nodes.items()}

    return fn
