"""Synthetic workloads of the BASELINE configs, generated on the device
(input harness, not product compute).

Mirrors the reference's synthetic producer: an axis-aligned box room with
solid interior boxes ray-cast by slab tests (_kernels/_numpy.py:29-47,
scenesim.py:145-163), log-normal depth noise with conf = 1/(1+|xi|) and a
per-decode scale gauge (backend.py:240-273), keyframe-buffer flushes of
"5 new + 1 old" frames (loops.py:89-111), landmark-tag descriptors with
sigma noise and 20% spurious rows (backend.py:283-311) rounded to
bf16-representable values, and pooled retrieval embeddings
(backend.py:216-226, database.py:78-80).  Everything is a pure function of
the seed (torch.Generator), so the CPU oracle can regenerate any slice.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch


@dataclass(frozen=True)
class SceneConfig:
    room: tuple = (8.0, 8.0, 4.0)
    boxes: tuple = (((1.0, 1.0, -2.0), (2.2, 2.0, -0.6)), ((-2.6, -1.0, -2.0), (-1.6, 0.4, 0.4)),
                    ((0.4, -3.0, -2.0), (1.4, -2.2, -1.0)))
    width: int = 518
    height: int = 392
    focal: float = 400.0
    depth_noise_sigma: float = 0.01
    gauge_range: tuple = (0.8, 1.25)
    radius: float = 2.0
    laps: float = 1.5


def intrinsics(cfg: SceneConfig):
    return np.array([cfg.focal, cfg.focal, (cfg.width - 1) / 2.0, (cfg.height - 1) / 2.0])


def _look_rotation(forward: np.ndarray) -> np.ndarray:
    """scenesim.look_rotation (world_from_cam, camera z along forward)."""
    z = forward / np.linalg.norm(forward)
    up = np.array([0.0, 0.0, 1.0])
    x = np.cross(up, z)
    x /= np.linalg.norm(x)
    y = np.cross(z, x)
    return np.stack([x, y, z], axis=1)


def _mat_to_quat(m):
    t = np.trace(m)
    if t > 0:
        r = math.sqrt(1.0 + t)
        s = 0.5 / r
        q = np.array([0.5 * r, (m[2, 1] - m[1, 2]) * s, (m[0, 2] - m[2, 0]) * s, (m[1, 0] - m[0, 1]) * s])
    else:
        i = int(np.argmax(np.diag(m)))
        j, k = (i + 1) % 3, (i + 2) % 3
        r = math.sqrt(1.0 + m[i, i] - m[j, j] - m[k, k])
        s = 0.5 / r
        q = np.empty(4)
        q[0] = (m[k, j] - m[j, k]) * s
        q[1 + i] = 0.5 * r
        q[1 + j] = (m[j, i] + m[i, j]) * s
        q[1 + k] = (m[k, i] + m[i, k]) * s
    return q / np.linalg.norm(q)


def trajectory(n: int, cfg: SceneConfig, seed: int = 0):
    """Circular keyframe trajectory (laps > 1 gives revisits) with a small
    height wobble: world_from_cam (R (n,3,3), t (n,3))."""
    rng = np.random.default_rng(seed)
    R = np.zeros((n, 3, 3))
    t = np.zeros((n, 3))
    for i in range(n):
        a = 2.0 * math.pi * cfg.laps * i / max(n - 1, 1)
        t[i] = [cfg.radius * math.cos(a), cfg.radius * math.sin(a), 0.15 * math.sin(3 * a)]
        fwd = np.array([-math.sin(a), math.cos(a), 0.05 * rng.normal()])
        R[i] = _look_rotation(fwd)
    return R, t


def raycast_depth(R: torch.Tensor, t: torch.Tensor, cfg: SceneConfig) -> torch.Tensor:
    """Perspective depth of frames (F,3,3)/(F,3) -> (F,H,W) float64, 0 = miss
    (first hit of room shell + solid boxes, _kernels/_numpy.py:29-47)."""
    dev = R.device
    F = R.shape[0]
    K = intrinsics(cfg)
    u = torch.arange(cfg.width, dtype=torch.float64, device=dev)
    v = torch.arange(cfg.height, dtype=torch.float64, device=dev)
    vv, uu = torch.meshgrid(v, u, indexing="ij")
    dcam = torch.stack([(uu - K[2]) / K[0], (vv - K[3]) / K[1], torch.ones_like(uu)], dim=-1)  # (H,W,3)
    out = torch.empty((F, cfg.height, cfg.width), dtype=torch.float64, device=dev)
    half = torch.tensor(cfg.room, dtype=torch.float64, device=dev) / 2
    shapes = [(-half, half)] + [(torch.tensor(a, dtype=torch.float64, device=dev),
                                 torch.tensor(b, dtype=torch.float64, device=dev)) for a, b in cfg.boxes]
    eps = 1e-9
    for f in range(F):
        d = dcam @ R[f].T  # world directions (H,W,3)
        o = t[f]
        with torch.no_grad():
            inv = 1.0 / d
            best = torch.full(d.shape[:2], float("inf"), dtype=torch.float64, device=dev)
            for bmin, bmax in shapes:
                t1 = (bmin - o) * inv
                t2 = (bmax - o) * inv
                near = torch.minimum(t1, t2).amax(-1)
                far = torch.maximum(t1, t2).amin(-1)
                ok = (near <= far) & (far > eps)
                hit = torch.where(near > eps, near, far)
                best = torch.where(ok, torch.minimum(best, hit), best)
            out[f] = torch.where(torch.isfinite(best), best, torch.zeros_like(best))
    return out


@dataclass
class SubmapBatch:
    """Decoded submaps of a run, ready for the FramePool."""

    frame_ids: list      # per submap tuple of keyframe ids (new..., old)
    depth: torch.Tensor  # (S, H, W) float32, S = total slots
    conf: torch.Tensor
    poses8: np.ndarray   # (S, 8) anchor_from_cam
    slot_offsets: list   # per submap first slot
    gauges: np.ndarray   # injected scales
    K4: np.ndarray


def flush_batches(n_keyframes: int, capacity: int = 5):
    """KeyframeBuffer flush sequence (loops.py:89-111): first batch holds
    capacity+1 new frames, then (capacity new, 1 old)."""
    out = []
    new, old = [], []
    for kf in range(n_keyframes):
        new.append(kf)
        if len(new) + len(old) > capacity:
            out.append(tuple(new) + tuple(old))
            new, old = [], [kf]
    return out


def make_submaps(n_keyframes: int, cfg: SceneConfig = SceneConfig(), seed: int = 0, device="cuda",
                 invalid_fraction: float = 0.0, batch_range=None) -> SubmapBatch:
    """Decoded submaps of a run of n_keyframes (synthetic decode, backend.py:228-281).
    batch_range=(b0, b1) decodes only those flush batches of the run (a
    rank's window of a sharded sequence); keyframe ids stay global."""
    Rw, tw = trajectory(n_keyframes, cfg, seed)
    batches = flush_batches(n_keyframes)
    if batch_range is not None:
        batches = batches[batch_range[0]:batch_range[1]]
    gen = torch.Generator(device=device)
    gen.manual_seed(1000 + seed)
    rng = np.random.default_rng(2000 + seed)
    S = sum(len(b) for b in batches)
    depth = torch.empty((S, cfg.height, cfg.width), dtype=torch.float32, device=device)
    conf = torch.empty_like(depth)
    poses8 = np.zeros((S, 8))
    offs, gauges = [], []
    Rd = torch.as_tensor(Rw, device=device)
    td = torch.as_tensor(tw, device=device)
    base_depth = {}
    s = 0
    for bi, b in enumerate(batches):
        offs.append(s)
        lo, hi = cfg.gauge_range
        scale = float(rng.uniform(lo, hi))
        gauges.append(scale)
        ids = list(b)
        need = [k for k in ids if k not in base_depth]
        if need:
            dd = raycast_depth(Rd[need], td[need], cfg)
            for k, d in zip(need, dd):
                base_depth[k] = d
        anchor = ids[0]
        Ra, ta = Rw[anchor], tw[anchor]
        for k in ids:
            d = base_depth[k] * scale
            xi = torch.randn(d.shape, generator=gen, device=device, dtype=torch.float64)
            d = d * torch.exp(cfg.depth_noise_sigma * xi)
            c = 1.0 / (1.0 + xi.abs())
            if invalid_fraction > 0:
                drop = torch.rand(d.shape, generator=gen, device=device) < invalid_fraction
                d = torch.where(drop, torch.zeros_like(d), d)
            c = torch.where(d > 0, c, torch.zeros_like(c))
            depth[s] = d.to(torch.float32)
            conf[s] = c.to(torch.float32)
            Rrel = Ra.T @ Rw[k]
            trel = Ra.T @ (tw[k] - ta) * scale
            poses8[s] = np.concatenate([[1.0], _mat_to_quat(Rrel), trel])
            s += 1
        # keep memory bounded: drop frames the next batch does not reference
        nxt = set(batches[bi + 1]) if bi + 1 < len(batches) else set()
        for k in list(base_depth):
            if k not in nxt:
                del base_depth[k]
    return SubmapBatch([tuple(b) for b in batches], depth, conf, poses8, offs, np.array(gauges), intrinsics(cfg))


def bf16_round(x: torch.Tensor) -> torch.Tensor:
    return x.to(torch.bfloat16).to(x.dtype)


def make_descriptor_pairs(n_pairs: int, n: int, m: int, d: int = 256, sigma: float = 0.05, spurious: float = 0.2,
                          seed: int = 0, device="cuda"):
    """(A_bits, B_bits, a_off, b_off): per pair, A = observed frame
    descriptors (tags + sigma noise, renormalised, `spurious` fresh rows),
    B = map tags (a random subset of size m); bf16-representable."""
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    A = torch.empty((n_pairs * n, d), dtype=torch.bfloat16, device=device)
    B = torch.empty((n_pairs * m, d), dtype=torch.bfloat16, device=device)
    for p in range(n_pairs):
        tags = torch.randn((max(n, m), d), generator=g, device=device, dtype=torch.float32)
        tags = tags / tags.norm(dim=1, keepdim=True)
        bmap = tags[torch.randperm(tags.shape[0], generator=g, device=device)[:m]]
        obs = tags[:n] + sigma * torch.randn((n, d), generator=g, device=device)
        spur = torch.rand(n, generator=g, device=device) < spurious
        fresh = torch.randn((n, d), generator=g, device=device)
        obs = torch.where(spur[:, None], fresh, obs)
        obs = obs / obs.norm(dim=1, keepdim=True)
        A[p * n:(p + 1) * n] = obs.to(torch.bfloat16)
        B[p * m:(p + 1) * m] = bmap.to(torch.bfloat16)
    a_off = np.arange(n_pairs + 1, dtype=np.int64) * n
    b_off = np.arange(n_pairs + 1, dtype=np.int64) * m
    return A.view(torch.int16), B.view(torch.int16), a_off, b_off


def make_descriptor_maps(n_frames: int, frames_per_map: int, n: int, m: int, d: int = 256, sigma: float = 0.05,
                         spurious: float = 0.2, seed: int = 0, device="cuda"):
    """Tracking workload with resident local maps: frame f is matched
    against map f // frames_per_map (tracking.py:173-194: consecutive frames
    of a keyframe interval see the same local map).  Returns (A_bits,
    B_bits, a_off, b_off, b_row) for tracking.match_batched_device: B holds
    each map once, b_off is the per-frame column prefix (m per frame) and
    b_row[f] the first row of frame f's map in B."""
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    n_maps = (n_frames + frames_per_map - 1) // frames_per_map
    A = torch.empty((n_frames * n, d), dtype=torch.bfloat16, device=device)
    B = torch.empty((n_maps * m, d), dtype=torch.bfloat16, device=device)
    for k in range(n_maps):
        tags = torch.randn((max(n, m), d), generator=g, device=device, dtype=torch.float32)
        tags = tags / tags.norm(dim=1, keepdim=True)
        B[k * m:(k + 1) * m] = tags[torch.randperm(tags.shape[0], generator=g, device=device)[:m]].to(torch.bfloat16)
        for f in range(k * frames_per_map, min(n_frames, (k + 1) * frames_per_map)):
            sel = torch.randperm(tags.shape[0], generator=g, device=device)[:n]
            obs = tags[sel] + sigma * torch.randn((n, d), generator=g, device=device)
            spur = torch.rand(n, generator=g, device=device) < spurious
            fresh = torch.randn((n, d), generator=g, device=device)
            obs = torch.where(spur[:, None], fresh, obs)
            A[f * n:(f + 1) * n] = (obs / obs.norm(dim=1, keepdim=True)).to(torch.bfloat16)
    a_off = np.arange(n_frames + 1, dtype=np.int64) * n
    b_off = np.arange(n_frames + 1, dtype=np.int64) * m
    b_row = (np.arange(n_frames, dtype=np.int64) // frames_per_map) * m
    return A.view(torch.int16), B.view(torch.int16), a_off, b_off, b_row


def pooled_embeddings(n: int, cfg: SceneConfig = SceneConfig(), dim: int = 64, tokens: int = 16,
                      noise: float = 0.02, seed: int = 0, device="cuda") -> torch.Tensor:
    """Pooled unit retrieval vectors of a keyframe run (backend.py:216-226:
    sqrt(2) cos(W f(pose) + b) + noise tokens; database.py:78-80 pooling)."""
    Rw, tw = trajectory(n, cfg, seed)
    rng = np.random.default_rng([seed, 404])
    Wm = rng.normal(size=(dim, 6))
    b = rng.uniform(0.0, 2.0 * math.pi, size=dim)
    feats = np.concatenate([tw / 2.0, Rw[:, :, 2]], axis=1)  # position / 2 m, viewing direction
    base = math.sqrt(2.0) * np.cos(feats @ Wm.T + b)
    tok = base[:, None, :] + noise * rng.normal(size=(n, tokens, dim))
    pooled = tok.mean(axis=1)
    pooled /= np.linalg.norm(pooled, axis=1, keepdims=True)
    return torch.as_tensor(pooled, device=device)


class DeviceDecoder:
    """SyntheticBackend.decode (backend.py:228-281) on the device, §8(f) rank 3.

    Wraps the reference's own SyntheticBackend (its world, trajectory,
    config, seed and decode-call counter): the gauge scale comes from the
    reference's own generator (default_rng([seed, 303, call_index]).uniform,
    backend.py:241-244, bit-exact), the relative poses are the reference's
    expressions (:265-266), and the frames are rendered and decoded by
    ec3r_synthetic_decode in one launch: render_depth's ray layout and BLAS
    FMA order, the bit-exact slab ray cast, log-normal depth noise with
    conf = 1/(1+|xi|), conf = 0 where depth <= 0.  The noise xi is a Philox
    stream (same distribution, different numbers than numpy's sequential
    ziggurat); with depth_noise_sigma = 0 the planes equal the reference's
    decode rounded to float32.  Depths / confidences come back as CUDA
    float32 tensors (the FramePool's format): DenseMapping.add_output takes
    them without a host copy."""

    DECODE_SALT = 303  # backend.py:33

    def __init__(self, backend, stream=None):
        self.b = backend
        self.stream = stream
        w = backend.world
        sol = [np.concatenate([np.asarray(w.room_min, float), np.asarray(w.room_max, float)])]
        for lo, hi in w.config.interior_boxes:
            sol.append(np.concatenate([np.asarray(lo, float), np.asarray(hi, float)]))
        self.solids = np.ascontiguousarray(np.stack(sol), np.float64)
        k = backend.intrinsics
        self.K4 = np.array([k.fx, k.fy, k.cx, k.cy], np.float64)

    def decode(self, embeddings):
        from . import _lib
        from .types import reference_module

        rb = reference_module("submap_slam.backend")
        rl = reference_module("submap_slam.liegroups")
        b, cfg = self.b, self.b.config
        if len(embeddings) < 2:
            raise rb.BatchTooSmall(f"decoder needs >= 2 embeddings, got {len(embeddings)}")
        if len(embeddings) > cfg.max_batch:
            raise rb.BatchTooLarge(f"decoder batch {len(embeddings)} exceeds max {cfg.max_batch}")
        frame_ids = tuple(int(getattr(e, "keyframe_id", e)) for e in embeddings)
        for fid in frame_ids:
            b._check_frame(fid)
        call_index = b._decode_calls
        b._decode_calls += 1
        rng = np.random.default_rng([b.seed, self.DECODE_SALT, call_index])
        lo, hi = cfg.gauge_scale_range
        scale = float(rng.uniform(lo, hi)) if hi > lo else float(lo)
        anchor = frame_ids[0]
        anchor_world = b.trajectory[anchor]
        k = b.intrinsics
        H, W = int(k.height), int(k.width)
        F = len(frame_ids)
        frames = np.zeros((F, 12), np.float64)
        poses = []
        for i, fid in enumerate(frame_ids):
            wc = b.trajectory[fid]
            frames[i, :9] = wc.rotation.matrix().reshape(-1)
            frames[i, 9:] = wc.translation
            rel = anchor_world.inverse().compose(wc)
            poses.append(rl.Pose3(rel.rotation, rel.translation * scale))
        dev = torch.device("cuda", torch.cuda.current_device())
        fr = torch.as_tensor(frames, device=dev)
        depth = torch.empty((F, H, W), dtype=torch.float32, device=dev)
        conf = torch.empty_like(depth)
        key = (int(b.seed) * 0x9E3779B97F4A7C15 + call_index * 0xBF58476D1CE4E5B9 + 0x94D049BB133111EB) % (1 << 64)
        _lib.check(_lib.lib().ec3r_synthetic_decode(self.solids.ctypes.data, len(self.solids), _lib.ptr(fr), F, H, W,
                                                    self.K4.ctypes.data, scale, float(cfg.depth_noise_sigma), key,
                                                    _lib.ptr(depth), _lib.ptr(conf), _lib.stream_ptr(self.stream)),
                   "ec3r_synthetic_decode")
        true_global = anchor_world.to_sim3().compose(rl.Sim3Transform(1.0 / scale, rl.Rotation3.identity(),
                                                                      np.zeros(3)))
        b.injected_gauges.append(rb.InjectedGauge(call_index, frame_ids, anchor, scale, true_global))
        return rb.ReconstructionOutput(frame_ids, depth, conf, tuple(poses), k, call_index)
