"""Drop-in for the stage-(a) producer interface of ``submap_slam.backend``:
``inverse_project`` (backend.py:78-101) runs in the K1 kernels
(csrc/project.cu) and returns a SubmapCloud whose float64 points are
bit-identical to the reference's.

``FramePool`` is the B200 data layout behind it: every decoded frame of every
submap stays resident in HBM as float32 depth + confidence planes
(n_slots, H, W) with its anchor_from_cam pose (float64), so registration
(K2/K3) and fusion (K4) stream the planes directly and the compacted cloud is
only materialised when host code asks for it.
"""

from __future__ import annotations

from typing import Optional

import numpy as np
import torch

from . import _lib
from .types import ReconstructionOutput, SubmapCloud, intrinsics_vec, sim3_to_vec


def _f32_dev(x) -> torch.Tensor:
    if isinstance(x, torch.Tensor):
        return x.to(device="cuda", dtype=torch.float32).contiguous()
    return torch.as_tensor(np.ascontiguousarray(np.asarray(x, dtype=np.float32)), device="cuda")


def inverse_project_device(depth: torch.Tensor, conf: torch.Tensor, K4, poses8: np.ndarray, frame_ids,
                           stream=None):
    """K1 on device planes.  depth/conf: (F,H,W) float32 (pool planes) or
    float64 (a reference output) CUDA; poses8: (F,8) host float64.  Returns
    device tensors (points (N,3) f64, conf (N,) f64, frame_ids (N,) i64,
    pixels (N,2) i64) trimmed to N (one D2H of N)."""
    L = _lib.lib()
    F, H, W = depth.shape
    total = F * H * W
    dev = depth.device
    pts = torch.empty((total, 3), dtype=torch.float64, device=dev)
    cf = torch.empty(total, dtype=torch.float64, device=dev)
    fid = torch.empty(total, dtype=torch.int64, device=dev)
    pix = torch.empty((total, 2), dtype=torch.int64, device=dev)
    n = torch.zeros(1, dtype=torch.int64, device=dev)
    ws_bytes = L.ec3r_inverse_project_workspace(F, H, W)
    ws = _lib.workspace(ws_bytes, dev, "ip")
    K4 = np.ascontiguousarray(np.asarray(K4, dtype=np.float64))
    P8 = np.ascontiguousarray(np.asarray(poses8, dtype=np.float64).reshape(F, 8))
    fids = np.ascontiguousarray(np.asarray(frame_ids, dtype=np.int64).reshape(F))
    if depth.dtype != conf.dtype or depth.dtype not in (torch.float32, torch.float64):
        raise ValueError("depth and confidence planes must both be float32 or both float64")
    fn = L.ec3r_inverse_project_f64 if depth.dtype == torch.float64 else L.ec3r_inverse_project
    _lib.check(fn(_lib.ptr(depth), _lib.ptr(conf), F, H, W, K4.ctypes.data, P8.ctypes.data, fids.ctypes.data,
                  _lib.ptr(pts), _lib.ptr(cf), _lib.ptr(fid), _lib.ptr(pix), _lib.ptr(n), _lib.ptr(ws), ws.numel(),
                  _lib.stream_ptr(stream)), "ec3r_inverse_project")
    N = int(n.item())
    return pts[:N], cf[:N], fid[:N], pix[:N]


def _dev_planes(x) -> torch.Tensor:
    """float32 inputs stay float32, everything else is consumed as float64
    (the reference's ReconstructionOutput dtype)."""
    if isinstance(x, torch.Tensor):
        dt = torch.float32 if x.dtype == torch.float32 else torch.float64
        return x.to(device="cuda", dtype=dt).contiguous()
    a = np.asarray(x)
    a = a if a.dtype == np.float32 else a.astype(np.float64)
    return torch.as_tensor(np.ascontiguousarray(a), device="cuda")


def inverse_project(output: ReconstructionOutput) -> SubmapCloud:
    """backend.py:78-101 — one 3D point per positive-depth pixel, in the
    submap frame, bit-identical to the reference's float64 result for the
    output's own depth dtype (float64 as decoded, or float32 planes)."""
    _lib.lib()
    F = len(output.frame_ids)
    if F == 0:
        return SubmapCloud(np.zeros((0, 3)), np.zeros(0), np.zeros(0, np.int64), np.zeros((0, 2), np.int64))
    depth = _dev_planes(output.depths)
    conf = _dev_planes(output.confidences)
    if depth.dtype != conf.dtype:
        depth, conf = depth.double(), conf.double()
    poses8 = np.stack([sim3_to_vec(p) for p in output.poses])
    pts, cf, fid, pix = inverse_project_device(depth, conf, intrinsics_vec(output.intrinsics), poses8,
                                               output.frame_ids)
    return SubmapCloud(pts.cpu().numpy(), cf.cpu().numpy(), fid.cpu().numpy(), pix.cpu().numpy())


class FramePool:
    """Resident frame planes in HBM (the B200 layout of decoded submaps).

    depth, conf: (capacity, H, W) float32 — one slot per decoded frame;
    poses: (capacity, 8) float64 anchor_from_cam of the slot's frame;
    globals: (capacity, 8) float64 world_from_anchor of the owning submap.
    Slots are allocated contiguously per submap; the pool doubles when full.
    """

    def __init__(self, height: int, width: int, K4, capacity: int = 64, device=None):
        _lib.lib()
        self.H, self.W = int(height), int(width)
        self.K4 = np.asarray(K4, dtype=np.float64).copy()
        self.device = torch.device("cuda") if device is None else torch.device(device)
        self.n = 0
        self._alloc(max(1, int(capacity)))

    def _alloc(self, cap: int):
        old = getattr(self, "depth", None)
        depth = torch.zeros((cap, self.H, self.W), dtype=torch.float32, device=self.device)
        conf = torch.zeros((cap, self.H, self.W), dtype=torch.float32, device=self.device)
        poses = torch.zeros((cap, 8), dtype=torch.float64, device=self.device)
        glob = torch.zeros((cap, 8), dtype=torch.float64, device=self.device)
        poses[:, 0] = 1.0
        poses[:, 1] = 1.0
        glob[:, 0] = 1.0
        glob[:, 1] = 1.0
        if old is not None and self.n:
            depth[: self.n] = self.depth[: self.n]
            conf[: self.n] = self.conf[: self.n]
            poses[: self.n] = self.poses[: self.n]
            glob[: self.n] = self.globals[: self.n]
        self.depth, self.conf, self.poses, self.globals = depth, conf, poses, glob
        self.capacity = cap

    def allocate(self, count: int) -> np.ndarray:
        if self.n + count > self.capacity:
            cap = self.capacity
            while cap < self.n + count:
                cap *= 2
            self._alloc(cap)
        slots = np.arange(self.n, self.n + count, dtype=np.int32)
        self.n += count
        return slots

    def write(self, slots, depths, confs, poses8):
        s0, s1 = int(slots[0]), int(slots[-1]) + 1
        assert s1 - s0 == len(slots), "slots of one submap are contiguous"
        self.depth[s0:s1].copy_(_f32_dev(depths).reshape(s1 - s0, self.H, self.W))
        self.conf[s0:s1].copy_(_f32_dev(confs).reshape(s1 - s0, self.H, self.W))
        self.poses[s0:s1].copy_(torch.as_tensor(np.asarray(poses8, np.float64).reshape(-1, 8), device=self.device))

    def set_global(self, slots, sim3_vec):
        s0, s1 = int(slots[0]), int(slots[-1]) + 1
        g = torch.as_tensor(np.asarray(sim3_vec, np.float64).reshape(1, 8), device=self.device)
        self.globals[s0:s1].copy_(g.expand(s1 - s0, 8))

    def nbytes(self) -> int:
        return 2 * self.n * self.H * self.W * 4


class LazyCloud:
    """SubmapCloud whose arrays are computed by K1 on first access (host code
    such as emit_corrections reads cloud.points; the dense path never does)."""

    def __init__(self, pool: FramePool, slots, frame_ids):
        self._pool = pool
        self._slots = np.asarray(slots)
        self._frame_ids = tuple(int(f) for f in frame_ids)
        self._host: Optional[SubmapCloud] = None
        self._dev = None

    def device_arrays(self):
        if self._dev is None:
            s0, s1 = int(self._slots[0]), int(self._slots[-1]) + 1
            P = self._pool
            poses8 = P.poses[s0:s1].cpu().numpy()
            self._dev = inverse_project_device(P.depth[s0:s1], P.conf[s0:s1], P.K4, poses8, self._frame_ids)
        return self._dev

    def materialize(self) -> SubmapCloud:
        if self._host is None:
            pts, cf, fid, pix = self.device_arrays()
            self._host = SubmapCloud(pts.cpu().numpy(), cf.cpu().numpy(), fid.cpu().numpy(), pix.cpu().numpy())
        return self._host

    @property
    def points(self):
        return self.materialize().points

    @property
    def confidences(self):
        return self.materialize().confidences

    @property
    def frame_ids(self):
        return self.materialize().frame_ids

    @property
    def pixels(self):
        return self.materialize().pixels
