"""Dense mapping on the B200 path: submap registration (stages a+b) and the
fused map (stage c), mirroring ``submap_slam.mapping`` (mapping.py:1-338).

* ``register_edges`` — every edge of a batch of submaps in ONE launch of the
  K2+K3 cluster kernel: pixel-identity correspondences on the shared
  keyframes (mapping.py:138-160), the min-count gate and the confidence floor
  (:174-179), weighted Umeyama (registration.py:38-102).
* ``DenseMapping`` — the reference's registration semantics (first submap
  fixed, strongest partner sets the global pose, edges T_ij; :190-211) on
  the resident ``FramePool``.
* ``VoxelMap`` / ``DenseMapping.fused_cloud(voxel=...)`` — K4 voxel-hash
  fusion (declared rule, oracle/fuse.py); ``voxel=None`` is the reference's
  plain concatenation (:332-338).
* ``b200_mapping_class(Mapping)`` — the drop-in: subclass of the reference
  ``Mapping`` whose dense path runs here.
"""

from __future__ import annotations

import os

import ctypes as C
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np
import torch

from . import _lib
from .backend import FramePool, LazyCloud
from .registration import raise_for_status
from .types import (NoSharedKeyframes, Sim3Transform, intrinsics_vec, sim3_to_vec, vec_to_sim3)


@dataclass
class DenseSubmap:
    """Submap (mapping.py:30-62) whose frames live in a FramePool."""

    id: int
    keyframe_ids: tuple
    slots: np.ndarray
    local_poses: dict
    intrinsics: object
    global_pose: Sim3Transform
    decode_call_index: int = -1
    cloud: object = None

    def keyframe_world_pose(self, kf_id):
        return self.global_pose.compose(self.local_poses[kf_id].to_sim3())


@dataclass(frozen=True, eq=False)
class MappingConfig:
    """mapping.py:65-71 (the dense-path knobs)."""

    confidence_floor_frac: float = 0.1
    min_correspondences: int = 10


@dataclass
class EdgeResult:
    status: int
    transform: Optional[Sim3Transform]
    rms: float
    count: int
    n_pairs: int


def edge_segments(sm, other):
    """Shared keyframes in sm.keyframe_ids order (mapping.py:145) as
    (slot in sm, slot in other) pairs."""
    segs = []
    oid = {kf: i for i, kf in enumerate(other.keyframe_ids)}
    for i, kf in enumerate(sm.keyframe_ids):
        j = oid.get(kf)
        if j is not None:
            segs.append((int(sm.slots[i]), int(other.slots[j])))
    return segs


def register_edges_device(pool: FramePool, seg_slots: torch.Tensor, edge_seg: torch.Tensor, n_edges: int,
                          floor_frac: float = 0.1, min_corr: int = 10, with_scale: bool = True,
                          keep_masks: Optional[torch.Tensor] = None, stream=None):
    """One launch of ec3r_register_edges; returns device tensors
    (sim3 (B,8), rms, count, npairs, status) without synchronizing."""
    L = _lib.lib()
    dev = pool.device
    sim3 = torch.empty((n_edges, 8), dtype=torch.float64, device=dev)
    rms = torch.empty(n_edges, dtype=torch.float64, device=dev)
    count = torch.empty(n_edges, dtype=torch.int64, device=dev)
    npairs = torch.empty(n_edges, dtype=torch.int64, device=dev)
    status = torch.empty(n_edges, dtype=torch.int32, device=dev)
    K4 = np.ascontiguousarray(pool.K4)
    _lib.check(L.ec3r_register_edges(_lib.ptr(pool.depth), _lib.ptr(pool.conf), pool.H, pool.W, K4.ctypes.data,
                                     _lib.ptr(pool.poses), _lib.ptr(seg_slots), _lib.ptr(edge_seg), n_edges,
                                     float(floor_frac), int(min_corr), int(bool(with_scale)), _lib.ptr(sim3),
                                     _lib.ptr(rms), _lib.ptr(count), _lib.ptr(npairs), _lib.ptr(status),
                                     _lib.ptr(keep_masks), None, 0, _lib.stream_ptr(stream)),
               "ec3r_register_edges")
    return sim3, rms, count, npairs, status


def register_edges(pool: FramePool, pairs: Sequence, config: MappingConfig = MappingConfig(),
                   with_keep_masks: bool = False):
    """Batched edges for a list of (sm, other) submap pairs.  Returns a list
    of EdgeResult (and the (n_seg, H, W) uint8 keep masks when asked)."""
    seg, eoff = [], [0]
    for sm, other in pairs:
        seg.extend(edge_segments(sm, other))
        eoff.append(len(seg))
    B = len(pairs)
    if B == 0:
        return ([], None) if with_keep_masks else []
    seg_t = torch.as_tensor(np.asarray(seg, np.int32).reshape(-1, 2), device=pool.device)
    eoff_t = torch.as_tensor(np.asarray(eoff, np.int32), device=pool.device)
    km = None
    if with_keep_masks:
        km = torch.zeros((max(len(seg), 1), pool.H, pool.W), dtype=torch.uint8, device=pool.device)
    sim3, rms, count, npairs, status = register_edges_device(pool, seg_t, eoff_t, B, config.confidence_floor_frac,
                                                             config.min_correspondences, True, km)
    sim3, rms, count, npairs, status = (x.cpu().numpy() for x in (sim3, rms, count, npairs, status))
    out = []
    for e in range(B):
        st = int(status[e])
        tr = vec_to_sim3(sim3[e]) if st == _lib.ST_OK else None
        out.append(EdgeResult(st, tr, float(rms[e]) if st == _lib.ST_OK else float("nan"), int(count[e]),
                              int(npairs[e])))
    if with_keep_masks:
        return out, km
    return out


class ChainPlan:
    """Device-resident plan for registering a run of submaps in order: the
    edges of every submap to its earlier partners (partners = submaps sharing
    a keyframe, mapping.py:164-169), their pixel segments, and the offsets
    the device pose chain (ec3r_chain_poses) walks."""

    def __init__(self, sms: Sequence[DenseSubmap], device="cuda"):
        self.sms = list(sms)
        index = {sm.id: i for i, sm in enumerate(self.sms)}
        owners: dict = {}
        pairs, partner, sub_edge_off = [], [], [0]
        for sm in self.sms:
            pids = {}
            for kf in sm.keyframe_ids:
                for sid in owners.get(kf, ()):
                    pids[sid] = None
            for sid in pids:
                pairs.append((sm, self.sms[index[sid]]))
                partner.append(index[sid])
            sub_edge_off.append(len(pairs))
            for kf in sm.keyframe_ids:
                owners.setdefault(kf, []).append(sm.id)
        self.pairs = pairs
        seg, eoff = [], [0]
        for a, b in pairs:
            seg.extend(edge_segments(a, b))
            eoff.append(len(seg))
        t = lambda x: torch.as_tensor(np.asarray(x, np.int32), device=device)  # noqa: E731
        self.seg = t(np.asarray(seg, np.int32).reshape(-1, 2))
        self.eoff = t(eoff)
        self.partner = t(partner if partner else [0])
        self.sub_edge_off = t(sub_edge_off)
        self.sub_slot_off = t(np.concatenate([[0], np.cumsum([len(sm.slots) for sm in self.sms])]))
        self.slot0 = int(self.sms[0].slots[0]) if self.sms else 0
        # the chain kernel writes slot globals through sub_slot_off from slot0:
        # the submaps' slots must be contiguous and in order
        if self.sms:
            all_slots = np.concatenate([np.asarray(sm.slots, np.int64) for sm in self.sms])
            if not np.array_equal(all_slots, np.arange(self.slot0, self.slot0 + all_slots.size)):
                raise ValueError("ChainPlan needs the submaps' pool slots contiguous and in registration order")
        self.n_edges = len(pairs)

    def run(self, pool: FramePool, config: MappingConfig = MappingConfig(), sub_globals: Optional[torch.Tensor] = None,
            stream=None):
        """Registration of every edge (one launch) + device pose chain (one
        launch) writing the pool's slot globals.  No host synchronisation.
        Returns (edge sim3, rms, count, npairs, status, sub_globals, sub_status)."""
        sim3, rms, count, npairs, status = register_edges_device(pool, self.seg, self.eoff, self.n_edges,
                                                                 config.confidence_floor_frac,
                                                                 config.min_correspondences, True, None, stream)
        S = len(self.sms)
        if sub_globals is None:
            sub_globals = torch.zeros((S, 8), dtype=torch.float64, device=pool.device)
            sub_globals[:, 0] = 1.0
            sub_globals[:, 1] = 1.0
        sub_status = torch.empty(S, dtype=torch.int32, device=pool.device)
        slot_globals = pool.globals[self.slot0:]
        _lib.check(_lib.lib().ec3r_chain_poses(_lib.ptr(sim3), _lib.ptr(count), _lib.ptr(status),
                                               _lib.ptr(self.partner), _lib.ptr(self.sub_edge_off), S,
                                               _lib.ptr(self.sub_slot_off), _lib.ptr(sub_globals),
                                               _lib.ptr(slot_globals), _lib.ptr(sub_status),
                                               _lib.stream_ptr(stream)), "ec3r_chain_poses")
        return sim3, rms, count, npairs, status, sub_globals, sub_status


class VoxelMap:
    """Owner of one ec3r_vhash handle (K4)."""

    def __init__(self, cell: float = 0.02, capacity: int = 1 << 20, stream=None, max_blocks: Optional[int] = None,
                 table_entries: int = 0):
        """capacity: voxels the emit can hold; max_blocks: 4x4x4 pool blocks
        (default capacity / 4; size it from a previous fill's n_blocks);
        table_entries: block-table size (0: 2x the pool)."""
        L = _lib.lib()
        self.cell = float(cell)
        h = C.c_void_p()
        if max_blocks is None:
            _lib.check(L.ec3r_vhash_create(C.byref(h), int(capacity), self.cell, _lib.stream_ptr(stream)),
                       "ec3r_vhash_create")
        else:
            _lib.check(L.ec3r_vhash_create_sized(C.byref(h), int(capacity), int(max_blocks), int(table_entries),
                                                 self.cell, _lib.stream_ptr(stream)), "ec3r_vhash_create_sized")
        self._h = h
        self.capacity = int(L.ec3r_vhash_capacity(h))  # voxel slots of the block pool
        self.expected = int(capacity)
        self._n = torch.zeros(1, dtype=torch.int64, device="cuda")

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value and _lib._lib is not None:
            try:
                torch.cuda.synchronize()
            except Exception:
                pass
            _lib._lib.ec3r_vhash_destroy(h)
            self._h = None

    @property
    def handle(self):
        return self._h

    def clear(self, stream=None):
        _lib.check(_lib.lib().ec3r_vhash_clear(self._h, _lib.stream_ptr(stream)), "ec3r_vhash_clear")

    def insert_frames(self, pool: FramePool, slots: torch.Tensor, stream=None):
        """slots: int32 CUDA tensor of pool slot ids."""
        K4 = np.ascontiguousarray(pool.K4)
        _lib.check(_lib.lib().ec3r_vhash_insert_frames(self._h, _lib.ptr(pool.depth), _lib.ptr(pool.conf), pool.H,
                                                       pool.W, K4.ctypes.data, _lib.ptr(pool.poses),
                                                       _lib.ptr(pool.globals), _lib.ptr(slots), int(slots.numel()),
                                                       _lib.stream_ptr(stream)), "ec3r_vhash_insert_frames")

    def insert_points(self, points: torch.Tensor, conf: torch.Tensor, sim3_vec, stream=None):
        g = np.ascontiguousarray(np.asarray(sim3_vec, np.float64))
        _lib.check(_lib.lib().ec3r_vhash_insert_points(self._h, _lib.ptr(points), _lib.ptr(conf),
                                                       int(points.shape[0]), g.ctypes.data,
                                                       _lib.stream_ptr(stream)), "ec3r_vhash_insert_points")

    def stats(self, stream=None) -> dict:
        s = _lib.VHashStats()
        _lib.check(_lib.lib().ec3r_vhash_stats_get(self._h, C.byref(s), _lib.stream_ptr(stream)),
                   "ec3r_vhash_stats_get")
        return dict(n_points_in=s.n_points_in, n_out_of_range=s.n_out_of_range, n_overflow=s.n_overflow,
                    n_slow_path=s.n_slow_path, n_blocks=s.n_blocks)

    def count(self, stream=None) -> int:
        """Number of fused voxels U (synchronises)."""
        _lib.check(_lib.lib().ec3r_vhash_count(self._h, _lib.ptr(self._n), _lib.stream_ptr(stream)),
                   "ec3r_vhash_count")
        return int(self._n.item())

    def stats_device(self, out: torch.Tensor, stream=None) -> torch.Tensor:
        """The stats() counters into a device int64[5] (no host round trip)."""
        _lib.check(_lib.lib().ec3r_vhash_stats_device(self._h, _lib.ptr(out), _lib.stream_ptr(stream)),
                   "ec3r_vhash_stats_device")
        return out

    def extract(self, sort: bool = True, stream=None, out=None, sync: bool = True):
        """Returns (keys int64, centroid (U,3) f32, wsum f32, count i32) CUDA
        tensors of length U (sorted by key when sort=True).  `out` may hold
        preallocated buffers of at least U rows.  sync=False (sorted only):
        no host read of U; returns the full `out` buffers plus the device
        int64[1] count instead -- check stats()["n_overflow"] == 0 afterwards
        (it also counts a map that outgrew the 32-bit sort keys a previous
        synced extract chose; re-run with sync=True then)."""
        L = _lib.lib()
        if out is None:
            if not sync:
                raise ValueError("extract(sync=False) needs preallocated out buffers")
            cap = self.count(stream)
            if cap == 0:  # an empty map (nothing valid was inserted): empty outputs, no emit
                return (torch.empty(0, dtype=torch.int64, device="cuda"),
                        torch.empty((0, 3), dtype=torch.float32, device="cuda"),
                        torch.empty(0, dtype=torch.float32, device="cuda"),
                        torch.empty(0, dtype=torch.int32, device="cuda"))
            out = (torch.empty(cap, dtype=torch.int64, device="cuda"),
                   torch.empty((cap, 3), dtype=torch.float32, device="cuda"),
                   torch.empty(cap, dtype=torch.float32, device="cuda"),
                   torch.empty(cap, dtype=torch.int32, device="cuda"))
        keys, cen, ws_, cnt = out
        wsb = L.ec3r_vhash_extract_workspace(self._h)
        ws = _lib.workspace(wsb, None, "vhash_extract")
        mode = (1 if sync else 2) if sort else 0
        _lib.check(L.ec3r_vhash_extract(self._h, _lib.ptr(keys), _lib.ptr(cen), _lib.ptr(ws_), _lib.ptr(cnt),
                                        _lib.ptr(self._n), mode, _lib.ptr(ws), ws.numel(),
                                        _lib.stream_ptr(stream)), "ec3r_vhash_extract")
        if sort and not sync:
            return keys, cen, ws_, cnt, self._n
        U = int(L.ec3r_vhash_extract_count(self._h)) if sort else -1
        if U < 0:
            U = int(self._n.item())
        return keys[:U], cen[:U], ws_[:U], cnt[:U]


# block-table entries per expected block for a re-sized map (sparse: fewer
# probe collisions at insert time; env override for A/B measurements)
TABLE_PER_BLOCK = int(os.environ.get("EC3R_TABLE_PER_BLOCK", "64"))


def fuse_slots(pool: FramePool, slots: torch.Tensor, cell: float, vmap: Optional[VoxelMap] = None,
               expected_voxels: Optional[int] = None, sort: bool = True, expected_blocks: Optional[int] = None):
    """Voxel fusion of pool slots with overflow-safe capacity growth.
    Returns (VoxelMap, (keys, centroid, wsum, count), stats).  With the
    expected voxel and block counts of a previous fill the map is sized at 2x
    both, with a sparse block table (64 entries per block: the insert speed
    of an oversized map, the clear and emit cost of a small one)."""
    if vmap is None or vmap.cell != cell:
        n_px = int(slots.numel()) * pool.H * pool.W
        cap = expected_voxels * 2 if expected_voxels else max(1 << 16, n_px // 8)
        vmap = VoxelMap(cell, cap, max_blocks=2 * expected_blocks if expected_blocks else None,
                        table_entries=TABLE_PER_BLOCK * expected_blocks if expected_blocks else 0)
    while True:
        vmap.clear()
        vmap.insert_frames(pool, slots)
        st = vmap.stats()
        if st["n_overflow"] == 0:
            out = vmap.extract(sort=sort)
            st = vmap.stats()  # the emit may overflow the voxel capacity too
            if st["n_overflow"] == 0:
                break
        vmap = VoxelMap(cell, vmap.expected * 4)  # default block sizing (capacity / 4)
    return vmap, out, st


class DenseMapping:
    """Resident dense map: FramePool + submaps + registration + fusion."""

    def __init__(self, height: int, width: int, intrinsics, config: MappingConfig = MappingConfig(),
                 slot_capacity: int = 64):
        self.intrinsics = intrinsics
        self.K4 = intrinsics_vec(intrinsics) if not isinstance(intrinsics, (list, tuple, np.ndarray)) \
            else np.asarray(intrinsics, np.float64)
        self.pool = FramePool(height, width, self.K4, slot_capacity)
        self.config = config
        self.submaps: dict[int, DenseSubmap] = {}
        self.pending: dict[int, DenseSubmap] = {}
        self.kf_submaps: dict[int, list] = {}  # keyframe -> submap ids (database.submap_ids)
        self.edges: list = []  # (i, j, T_ij, info)
        self._next_id = 0
        self._vmap: Optional[VoxelMap] = None
        self._last_voxels: Optional[int] = None

    # -- submap construction (mapping.py:114-136) --------------------------
    def add_submap(self, frame_ids, depths, confs, poses, call_index: int = -1) -> DenseSubmap:
        F = len(frame_ids)
        slots = self.pool.allocate(F)
        poses8 = np.stack([sim3_to_vec(p) if not isinstance(p, np.ndarray) else np.asarray(p, float)
                           for p in poses])
        self.pool.write(slots, depths, confs, poses8)
        local = {}
        for k, fid in enumerate(frame_ids):
            local[int(fid)] = poses[k] if not isinstance(poses[k], np.ndarray) else None
        sm = DenseSubmap(self._next_id, tuple(int(f) for f in frame_ids), slots, local, self.intrinsics,
                         Sim3Transform.identity(), call_index)
        sm.cloud = LazyCloud(self.pool, slots, sm.keyframe_ids)
        self._next_id += 1
        return sm

    def add_output(self, output) -> DenseSubmap:
        """From a reference ReconstructionOutput (backend.py:51-58)."""
        return self.add_submap(output.frame_ids, output.depths, output.confidences, output.poses,
                               output.call_index)

    # -- registration (mapping.py:162-211) ---------------------------------
    def partners(self, sm) -> list:
        out: dict = {}
        for kf in sm.keyframe_ids:
            for sid in self.kf_submaps.get(kf, ()):
                if sid != sm.id:
                    out[sid] = None
        return list(out)

    def registration_edges(self, sm, partner_ids=None):
        """mapping.py:162-188 for one submap (one launch over its partners)."""
        pids = self.partners(sm) if partner_ids is None else partner_ids
        res = register_edges(self.pool, [(sm, self.submaps[s]) for s in pids], self.config)
        return self._edges_from(sm, pids, res)

    def _edges_from(self, sm, pids, res):
        edges = []
        for sid, r in zip(pids, res):
            if r.status == _lib.ST_SKIP:
                continue
            raise_for_status(r.status, r.count)  # align_point_sets raises out of the loop
            info = np.eye(7) * (r.count / (1.0 + r.rms * r.rms))
            edges.append((sid, r.transform, info, r.count, r.rms))
        if not edges:
            raise NoSharedKeyframes(f"submap {sm.id} shares no usable keyframes with existing submaps")
        return edges

    def _commit(self, sm):
        self.submaps[sm.id] = sm
        self.pool.set_global(sm.slots, sim3_to_vec(sm.global_pose))
        for kf in sm.keyframe_ids:
            lst = self.kf_submaps.setdefault(kf, [])
            if sm.id not in lst:
                lst.append(sm.id)

    def forget(self, sm):
        """Drop a submap from the map (its pool slots stay allocated): used
        for the halo stub of a sharded window (dist.register_window)."""
        self.submaps.pop(sm.id, None)
        for kf in sm.keyframe_ids:
            lst = self.kf_submaps.get(kf, [])
            if sm.id in lst:
                lst.remove(sm.id)

    def register_submap(self, sm):
        """mapping.py:190-211."""
        if not self.submaps:
            sm.global_pose = Sim3Transform.identity()
            self._commit(sm)
            return 0
        edges = self.registration_edges(sm)
        best = max(edges, key=lambda e: e[3])
        sm.global_pose = self.submaps[best[0]].global_pose.compose(best[1])
        self._commit(sm)
        for sid, tr, info, _, _ in edges:
            self.edges.append((sid, sm.id, tr, info))
        return len(edges)

    def register_chain(self, sms: Sequence[DenseSubmap]):
        """Register submaps in order with ALL their edges in one launch.
        Equivalent to calling register_submap on each in turn (edge
        measurements do not depend on global poses)."""
        pending = list(sms)
        kf_map = {k: list(v) for k, v in self.kf_submaps.items()}
        pairs, spans, pid_lists = [], [], []
        first_fixed = not self.submaps
        for idx, sm in enumerate(pending):
            if idx == 0 and first_fixed:
                spans.append((0, 0))
                pid_lists.append([])
            else:
                pids = {}
                for kf in sm.keyframe_ids:
                    for sid in kf_map.get(kf, ()):
                        if sid != sm.id:
                            pids[sid] = None
                pids = list(pids)
                spans.append((len(pairs), len(pairs) + len(pids)))
                pid_lists.append(pids)
                lookup = {**self.submaps, **{p.id: p for p in pending[:idx]}}
                pairs.extend((sm, lookup[s]) for s in pids)
            for kf in sm.keyframe_ids:
                kf_map.setdefault(kf, []).append(sm.id)
        res = register_edges(self.pool, pairs, self.config)
        n_edges = 0
        for idx, sm in enumerate(pending):
            if idx == 0 and first_fixed:
                sm.global_pose = Sim3Transform.identity()
                self._commit(sm)
                continue
            a, b = spans[idx]
            edges = self._edges_from(sm, pid_lists[idx], res[a:b])
            best = max(edges, key=lambda e: e[3])
            sm.global_pose = self.submaps[best[0]].global_pose.compose(best[1])
            self._commit(sm)
            for sid, tr, info, _, _ in edges:
                self.edges.append((sid, sm.id, tr, info))
            n_edges += len(edges)
        return n_edges

    # -- fused map (mapping.py:332-338 + declared voxel rule) ---------------
    def all_slots(self) -> torch.Tensor:
        sl = np.concatenate([sm.slots for sm in self.submaps.values()]) if self.submaps else np.zeros(0, np.int32)
        return torch.as_tensor(sl.astype(np.int32), device=self.pool.device)

    def fused_cloud(self, voxel: Optional[float] = None, sort: bool = True):
        """voxel=None: (points (N,3) f64, conf (N,)) numpy, the reference's
        concatenation bit-for-bit.  voxel=cell: dict of numpy arrays keys /
        centroid / wsum / count (sorted by key) from the voxel hash."""
        if voxel is None:
            pts, cfs = [], []
            L = _lib.lib()
            for sm in self.submaps.values():
                p, c, _, _ = sm.cloud.device_arrays()
                out = torch.empty_like(p)
                g = np.ascontiguousarray(sim3_to_vec(sm.global_pose))
                _lib.check(L.ec3r_sim3_apply(_lib.ptr(p), int(p.shape[0]), g.ctypes.data, _lib.ptr(out),
                                             _lib.stream_ptr()), "ec3r_sim3_apply")
                pts.append(out)
                cfs.append(c)
            if not pts:
                return np.zeros((0, 3)), np.zeros(0)
            return torch.cat(pts).cpu().numpy(), torch.cat(cfs).cpu().numpy()
        self._vmap, (k, c, w, n), st = fuse_slots(self.pool, self.all_slots(), float(voxel), self._vmap,
                                                  self._last_voxels, sort)
        self._last_voxels = int(k.numel())
        return dict(keys=k.cpu().numpy(), centroid=c.cpu().numpy(), wsum=w.cpu().numpy(), count=n.cpu().numpy(),
                    stats=st)


def b200_mapping_class(base):
    """Drop-in subclass of the reference ``submap_slam.mapping.Mapping``:
    build_submap keeps the decoded planes resident, _shared_correspondences /
    _registration_edges run through the batched K2+K3 kernel, fused_cloud
    gains ``voxel=``.  Host bookkeeping (database, pose graph, corrections,
    loop mapping) is the reference's own code."""

    class B200Mapping(base):
        def __init__(self, backend, config=None, slot_capacity: int = 64):
            super().__init__(backend) if config is None else super().__init__(backend, config)
            self._dense: Optional[DenseMapping] = None
            self._slot_capacity = slot_capacity
            self._dense_sm: dict = {}

        def _ensure(self, output):
            if self._dense is None:
                k = output.intrinsics
                cfg = MappingConfig(self.config.confidence_floor_frac, self.config.min_correspondences)
                self._dense = DenseMapping(k.height, k.width, k, cfg, self._slot_capacity)
            return self._dense

        def build_submap(self, batch):
            from .types import ReconstructionOutput  # noqa: F401
            ids = batch.ordered()
            if len(ids) < 2:
                raise ValueError("flush batch needs at least 2 keyframes")
            from submap_slam.errors import MissingEmbedding
            for kf in batch.old_ids:
                if not self.database.has_embedding(kf):
                    raise MissingEmbedding(f"old keyframe {kf} missing from the database")
            embeddings = self.embeddings_for(ids)
            output = self.backend.decode(embeddings)
            dm = self._ensure(output)
            dsm = dm.add_output(output)
            from submap_slam.mapping import Submap
            sm = Submap(id=self._next_submap_id, keyframe_ids=tuple(ids), cloud=dsm.cloud,
                        local_poses={fid: output.poses[k] for k, fid in enumerate(output.frame_ids)},
                        intrinsics=output.intrinsics, global_pose=Sim3Transform.identity(),
                        decode_call_index=output.call_index)
            dsm.id = sm.id
            self._dense_sm[sm.id] = dsm
            self._next_submap_id += 1
            return sm

        def _registration_edges(self, sm):
            partners: dict = {}
            for kf in sm.keyframe_ids:
                if kf in self.database:
                    for sid in self.database.get(kf).submap_ids:
                        if sid != sm.id:
                            partners[sid] = None
            pids = list(partners)
            dm = self._dense
            dsm = self._dense_sm[sm.id]
            res = register_edges(dm.pool, [(dsm, self._dense_sm[s]) for s in pids], dm.config)
            return dm._edges_from(sm, pids, res)

        def _commit(self, sm, fixed):
            super()._commit(sm, fixed)
            dsm = self._dense_sm[sm.id]
            dsm.global_pose = sm.global_pose
            self._dense.pool.set_global(dsm.slots, sim3_to_vec(sm.global_pose))

        def optimize(self):
            rep = super().optimize()
            for sid, sm in self.submaps.items():
                self._dense_sm[sid].global_pose = sm.global_pose
                self._dense.pool.set_global(self._dense_sm[sid].slots, sim3_to_vec(sm.global_pose))
            return rep

        def fused_cloud(self, voxel=None):
            dm = self._dense
            if dm is None:
                return super().fused_cloud()
            dm.submaps = {sid: self._dense_sm[sid] for sid in self.submaps}
            return dm.fused_cloud(voxel)

    return B200Mapping
