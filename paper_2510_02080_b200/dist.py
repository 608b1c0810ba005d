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
    """Owner-partitioned global voxel map from per-rank local maps: the
    partials of a rank's local VoxelMap are bucketed by owner on the device
    (ec3r_vhash_extract_partials), exchanged in one all-to-all and merged
    into this rank's owned map (ec3r_vhash_merge_partials), whose sorted
    emit is the rank's partition of the global map.  Buffers and the owned
    map persist across calls (no allocation in steady state)."""

    def __init__(self, cell: float, group=None):
        self.cell = float(cell)
        self.group = group
        self.rank, self.world = _world(group)
        self.owned = None
        self._buf = None
        self.out = None

    def _buffers(self, n: int):
        if self._buf is None or self._buf[0].shape[0] < n:
            m = max(n, 1)
            self._buf = (torch.empty(m, dtype=torch.int64, device="cuda"),
                         torch.empty((m, 4), dtype=torch.float32, device="cuda"),
                         torch.empty(m, dtype=torch.int32, device="cuda"),
                         torch.zeros(self.world, dtype=torch.int64, device="cuda"))
        return self._buf

    def run(self, local, n_local: int, stream=None):
        """local: this rank's fused VoxelMap holding n_local voxels."""
        from . import _lib
        from .mapping import VoxelMap

        L = _lib.lib()
        keys, sums4, cnt, rank_counts = self._buffers(n_local)
        rank_counts.zero_()
        wsb = L.ec3r_vhash_extract_workspace(local.handle) + 1024
        ws = _lib.workspace(wsb, keys.device, "partials")
        _lib.check(L.ec3r_vhash_extract_partials(local.handle, self.world, _lib.ptr(keys), _lib.ptr(sums4),
                                                 _lib.ptr(cnt), _lib.ptr(rank_counts), _lib.ptr(ws), ws.numel(),
                                                 _lib.stream_ptr(stream)), "ec3r_vhash_extract_partials")
        rk, rs, rcnt = exchange_partials(keys, sums4, cnt, rank_counts.tolist(), self.group)
        n = int(rk.shape[0])
        while True:  # grow until neither the merge nor the emit overflows
            if self.owned is None or self.owned.expected < n:
                self.owned = VoxelMap(self.cell, capacity=max(2 * n, 1 << 16))
            self.owned.clear(stream)
            if n:
                _lib.check(L.ec3r_vhash_merge_partials(self.owned.handle, _lib.ptr(rk), _lib.ptr(rs),
                                                       _lib.ptr(rcnt), n, _lib.stream_ptr(stream)),
                           "ec3r_vhash_merge_partials")
            if self.owned.stats(stream)["n_overflow"] == 0:
                if self.out is None or self.out[0].shape[0] < n:
                    self.out = (torch.empty(max(n, 1), dtype=torch.int64, device="cuda"),
                                torch.empty((max(n, 1), 3), dtype=torch.float32, device="cuda"),
                                torch.empty(max(n, 1), dtype=torch.float32, device="cuda"),
                                torch.empty(max(n, 1), dtype=torch.int32, device="cuda"))
                res = self.owned.extract(sort=True, stream=stream, out=self.out)
                if self.owned.stats(stream)["n_overflow"] == 0:
                    return res
            self.owned = VoxelMap(self.cell, capacity=4 * max(self.owned.expected, 2 * n))


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
    # round 2 (forwards): header (count, ids) then the frames
    send = []
    if rank + 1 < world:
        wanted = {int(x) for x in want.tolist() if x >= 0}
        last = window[-1]
        pick = [k for k, f in enumerate(last.keyframe_ids) if f in wanted]
        hdr = torch.full((1 + HALO_MAX,), -1, **i64)
        hdr[0] = len(pick)
        hdr[1: 1 + len(pick)] = torch.tensor([last.keyframe_ids[k] for k in pick], dtype=torch.int64)
        sl = torch.as_tensor(np.asarray(last.slots, np.int64)[pick], device=dev)
        send = [hdr, pool.depth.index_select(0, sl).to(tdev), pool.conf.index_select(0, sl).to(tdev),
                pool.poses.index_select(0, sl).to(tdev)]
        n_send = len(pick)
    hdr_in = torch.full((1 + HALO_MAX,), -1, **i64)
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
    ids = [int(x) for x in hdr_in[1: 1 + n_in].tolist()]
    return mapping.add_submap(ids, recv[0].to(dev), recv[1].to(dev), list(recv[2].cpu().numpy()))


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
    mapping.register_chain(([stub] if stub is not None else []) + list(window))
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
