"""Drop-in for the global-retrieval scoring of ``submap_slam.loops``
(update_similarity, loops.py:184-243) on the B200 path (K6,
csrc/retrieval.cu).

The GPU scores the strided coarse grid and the refinement windows in float64
and emits them in the reference's emission order; the host applies only the
stateful parts of the reference — the similarity-matrix cache
(loops.py:201-210) and the admitted-once set kept on the matrix
(loops.py:212-216, 240-242).  ``RetrievalDB`` keeps the pooled vectors
resident for repeated calls and shards the coarse rows across ranks.
"""

from __future__ import annotations

from typing import Optional

import numpy as np
import torch

from . import _lib


class SimilarityMatrix:
    """loops.py:156-176 (used when the reference class is not at hand)."""

    def __init__(self):
        self._scores: dict = {}

    @staticmethod
    def _key(a, b):
        return (a, b) if a <= b else (b, a)

    def set(self, a, b, score):
        self._scores[self._key(a, b)] = score

    def get(self, a, b):
        return self._scores.get(self._key(a, b))

    def __len__(self):
        return len(self._scores)

    def items(self):
        return self._scores.items()


_cap_cache: dict = {}  # (K, stride, k_begin, k_end) -> refinement capacity that sufficed


def retrieval_device(pooled: torch.Tensor, stride: int, exclusion: int, tau_g: float, tau_l: float,
                     k_begin: int = 0, k_end: int = -1, cap_refine: int = 1 << 16, stream=None):
    """Run K6 on a (K, D) float64 CUDA tensor.  Returns numpy arrays
    (coarse_pairs, coarse_scores, cand_pairs, cand_scores, eval_pairs,
    eval_scores) of ORDER indices, growing capacities until nothing is
    truncated."""
    L = _lib.lib()
    K, D = pooled.shape
    dev = pooled.device
    Kc = (K + stride - 1) // stride
    kb = max(0, k_begin)
    ke = Kc if k_end is None or k_end < 0 or k_end > Kc else k_end
    rows = max(ke - kb, 0)
    R = (2 * stride - 1) ** 2
    key = (int(K), int(stride), kb, ke)
    cap_refine = max(int(cap_refine), _cap_cache.get(key, 0))  # start from the last call's need
    while True:
        cap_c = max(rows * Kc, 1)
        cp = torch.empty((cap_c, 2), dtype=torch.int32, device=dev)
        cs = torch.empty(cap_c, dtype=torch.float64, device=dev)
        qp = torch.empty((cap_refine, 2), dtype=torch.int32, device=dev)
        qs = torch.empty(cap_refine, dtype=torch.float64, device=dev)
        ep = torch.empty((cap_refine, 2), dtype=torch.int32, device=dev)
        es = torch.empty(cap_refine, dtype=torch.float64, device=dev)
        counts = torch.zeros(4, dtype=torch.int64, device=dev)
        wsb = L.ec3r_retrieval_workspace(K, stride, cap_refine)
        ws = _lib.workspace(wsb, dev, "retrieval")
        _lib.check(L.ec3r_retrieval(_lib.ptr(pooled), K, D, stride, exclusion, float(tau_g), float(tau_l),
                                    _lib.ptr(cp), _lib.ptr(cs), _lib.ptr(qp), _lib.ptr(qs), _lib.ptr(ep),
                                    _lib.ptr(es), cap_refine, _lib.ptr(counts), kb, ke, _lib.ptr(ws), ws.numel(),
                                    _lib.stream_ptr(stream)), "ec3r_retrieval")
        n_c, n_q, n_e, n_h = (int(x) for x in counts.cpu())
        if n_q <= cap_refine and n_e <= cap_refine and n_h <= cap_refine // R + 1:
            break
        cap_refine = max(cap_refine * 4, (n_h + 1) * R, n_e)
    _cap_cache[key] = cap_refine
    outs = (cp[:n_c], cs[:n_c], qp[:n_q], qs[:n_q], ep[:n_e], es[:n_e])
    return tuple(_to_host(x) for x in outs) if outs[0].is_cuda else tuple(x.numpy() for x in outs)


# Margin guard.  The device scores with a sequential fma dot, the reference
# with numpy's BLAS ddot (loops.py:205): the two agree to a few ulps
# (|error| <= D * 2^-52 * sum|a_k b_k| ~ 1e-14 for unit vectors), so only a
# score within GUARD_BAND of tau_global / tau_local can be decided
# differently.  Those pairs are re-scored on the host with the reference's
# own expression, float(pa @ pb), and every decision is taken on that score.
GUARD_BAND = 1e-12
_guard_stats = {"coarse_rescored": 0, "refine_rescored": 0, "coarse_flips": 0, "refine_flips": 0}


def last_guard_stats() -> dict:
    return dict(_guard_stats)


def _window_pairs(a: int, b: int, stride: int, exclusion: int, K: int):
    """Refinement window of a coarse hit in the reference's order
    (loops.py:228-238): (da, db) ascending, in bounds, outside exclusion."""
    out = []
    for da in range(-(stride - 1), stride):
        for db in range(-(stride - 1), stride):
            ia, ib = a + da, b + db
            if 0 <= ia < K and 0 <= ib < K and abs(ia - ib) >= exclusion:
                out.append((ia, ib))
    return out


def guard_retrieval(host_pooled: np.ndarray, outs, stride: int, exclusion: int, tau_g: float, tau_l: float,
                    band: float = GUARD_BAND):
    """Apply the margin guard to retrieval_device's lists (ORDER indices).
    host_pooled: (K, D) float64, the vectors the reference multiplies."""
    cp, cs, qp, qs, ep, es = outs
    for k in _guard_stats:
        _guard_stats[k] = 0
    P = host_pooled
    K = P.shape[0]

    def rescore(pairs):
        return np.array([float(P[i] @ P[j]) for i, j in pairs], dtype=np.float64)

    near = np.flatnonzero(np.abs(cs - tau_g) < band)
    flips = []
    if near.size:
        cs = cs.copy()
        old = cs[near] > tau_g
        cs[near] = rescore(cp[near])
        _guard_stats["coarse_rescored"] = int(near.size)
        flips = near[(cs[near] > tau_g) != old].tolist()
        _guard_stats["coarse_flips"] = len(flips)
    if flips:
        # rebuild the refinement groups in coarse emission order: unchanged
        # hits keep the device's scored group, flipped-in hits are scored here
        dev_hits = np.flatnonzero(np.where(np.isin(np.arange(len(cs)), flips), ~(cs > tau_g), cs > tau_g))
        sizes = [len(_window_pairs(int(cp[h, 0]), int(cp[h, 1]), stride, exclusion, K)) for h in dev_hits]
        groups = dict(zip(dev_hits.tolist(), np.split(np.arange(len(ep)), np.cumsum(sizes)[:-1]) if sizes else []))
        new_p, new_s = [], []
        for h in np.flatnonzero(cs > tau_g).tolist():
            if h in groups:
                idx = groups[h]
                new_p.append(ep[idx])
                new_s.append(es[idx])
            else:
                w = _window_pairs(int(cp[h, 0]), int(cp[h, 1]), stride, exclusion, K)
                new_p.append(np.asarray(w, np.int32).reshape(-1, 2))
                new_s.append(rescore(w))
        ep = np.concatenate(new_p) if new_p else np.zeros((0, 2), np.int32)
        es = np.concatenate(new_s) if new_s else np.zeros(0)
    near_r = np.flatnonzero(np.abs(es - tau_l) < band)
    if near_r.size:
        es = es.copy()
        old = es[near_r] > tau_l
        es[near_r] = rescore(ep[near_r])
        _guard_stats["refine_rescored"] = int(near_r.size)
        _guard_stats["refine_flips"] = int(((es[near_r] > tau_l) != old).sum())
    if flips or near_r.size:
        keep = es > tau_l
        qp, qs = ep[keep], es[keep]
    return cp, cs, qp, qs, ep, es


_pinned: dict = {}


def _to_host(t: torch.Tensor) -> np.ndarray:
    """D2H through a cached pinned buffer (pageable copies of the multi-MB
    lists ran at ~3.5 GB/s)."""
    n = t.numel() * t.element_size()
    buf = _pinned.get(t.dtype)
    if buf is None or buf.numel() < t.numel():
        buf = torch.empty(max(t.numel(), 1 << 16), dtype=t.dtype, pin_memory=True)
        _pinned[t.dtype] = buf
    view = buf[: t.numel()]
    if n:
        view.copy_(t.reshape(-1), non_blocking=True)
        torch.cuda.current_stream(t.device).synchronize()
    return view.numpy().reshape(t.shape).copy()


def _populate(matrix, kfs: np.ndarray, pairs: np.ndarray, scores: np.ndarray):
    if len(pairs) == 0:
        return
    a = kfs[pairs[:, 0]]
    b = kfs[pairs[:, 1]]
    lo = np.minimum(a, b).tolist()
    hi = np.maximum(a, b).tolist()
    store = getattr(matrix, "_scores", None)
    if isinstance(store, dict):
        store.update(zip(zip(lo, hi), scores.tolist()))
    else:
        for x, y, s in zip(lo, hi, scores.tolist()):
            matrix.set(x, y, s)


def admit(matrix, kfs: np.ndarray, cand_pairs: np.ndarray, cand_scores: np.ndarray):
    """Admitted-once rule (loops.py:212-216, 240-242) over candidates in
    emission order; the set lives on the matrix like the reference's."""
    seen = getattr(matrix, "_admitted", None)
    if seen is None:
        seen = set()
        matrix._admitted = seen
    out = []
    a = kfs[cand_pairs[:, 0]].tolist() if len(cand_pairs) else []
    b = kfs[cand_pairs[:, 1]].tolist() if len(cand_pairs) else []
    for x, y, s in zip(a, b, cand_scores.tolist()):
        key = (x, y) if x <= y else (y, x)
        if key not in seen:
            seen.add(key)
            out.append((key, s))
    return out


def update_similarity(matrix, database, stride: int, cfg) -> list:
    """loops.py:184-243 — extend the similarity matrix; returns pairs newly
    over tau_local, in the reference's emission order."""
    _lib.lib()
    order = [kf for kf in database.ids_in_order() if database.get(kf).pooled is not None]
    if not order:
        return []
    pooled = torch.as_tensor(np.stack([np.asarray(database.get(kf).pooled, np.float64) for kf in order]),
                             device="cuda")  # the host stack is kept for the margin guard
    kfs = np.asarray(order, dtype=np.int64)
    host = np.stack([np.asarray(database.get(kf).pooled, np.float64) for kf in order])
    outs = retrieval_device(pooled, int(stride), int(cfg.exclusion_zone()), float(cfg.tau_global),
                            float(cfg.tau_local))
    cp, cs, qp, qs, ep, es = guard_retrieval(host, outs, int(stride), int(cfg.exclusion_zone()),
                                             float(cfg.tau_global), float(cfg.tau_local))
    _populate(matrix, kfs, cp, cs)
    _populate(matrix, kfs, ep, es)
    return admit(matrix, kfs, qp, qs)


class RetrievalDB:
    """Resident pooled-vector database (database.py:72-80 pooled vectors in
    insertion order) for repeated / sharded retrieval."""

    def __init__(self, dim: int, capacity: int = 1024, device=None):
        self.device = torch.device("cuda") if device is None else torch.device(device)
        self.dim = int(dim)
        self.vec = torch.zeros((capacity, self.dim), dtype=torch.float64, device=self.device)
        self.kf = np.zeros(capacity, dtype=np.int64)
        self.host = np.zeros((capacity, self.dim), dtype=np.float64)  # margin-guard copy (host side of append)
        self.n = 0

    def append(self, kf_ids, pooled):
        pooled_h = np.asarray(pooled, np.float64).reshape(-1, self.dim)
        pooled = torch.as_tensor(pooled_h, device=self.device)
        k = pooled.shape[0]
        if self.n + k > self.vec.shape[0]:
            cap = self.vec.shape[0]
            while cap < self.n + k:
                cap *= 2
            v = torch.zeros((cap, self.dim), dtype=torch.float64, device=self.device)
            v[: self.n] = self.vec[: self.n]
            self.vec = v
            kf = np.zeros(cap, np.int64)
            kf[: self.n] = self.kf[: self.n]
            self.kf = kf
            hv = np.zeros((cap, self.dim), np.float64)
            hv[: self.n] = self.host[: self.n]
            self.host = hv
        self.vec[self.n:self.n + k] = pooled
        self.host[self.n:self.n + k] = pooled_h
        self.kf[self.n:self.n + k] = np.asarray(kf_ids, np.int64)
        self.n += k

    def score(self, stride: int, exclusion: int, tau_g: float, tau_l: float, k_begin: int = 0, k_end: int = -1,
              guard: bool = True):
        outs = retrieval_device(self.vec[: self.n], stride, exclusion, tau_g, tau_l, k_begin, k_end)
        if not guard:
            return outs
        return guard_retrieval(self.host[: self.n], outs, stride, exclusion, tau_g, tau_l)

    def update(self, matrix, stride: int, cfg, k_begin: int = 0, k_end: int = -1) -> list:
        cp, cs, qp, qs, ep, es = self.score(stride, cfg.exclusion_zone(), cfg.tau_global, cfg.tau_local,
                                            k_begin, k_end)
        kfs = self.kf[: self.n]
        _populate(matrix, kfs, cp, cs)
        _populate(matrix, kfs, ep, es)
        return admit(matrix, kfs, qp, qs)


# ---------------------------------------------------------------------------
# Local loop candidates (loops.py:114-133; K8, csrc/local_cand.cu)

def local_candidates_device(positions: torch.Tensor, world_from_cam: torch.Tensor, intrinsics, tau_p: float,
                            stream=None, ambiguous: bool = False, amb_cap: int = 4096):
    """Projection counts of the map points (N, 3) float64 into K keyframes
    (world_from_cam: (K, 8) float64 {s, q, t}) in one launch.  Returns
    (counts (K,) int64, candidate (K,) int32) CUDA tensors; intrinsics =
    (fx, fy, cx, cy, width, height).  ambiguous=True also returns the
    margin-guard list (n, 3) int32 numpy (keyframe, point, device decision)."""
    L = _lib.lib()
    pts = positions.reshape(-1, 3).to(torch.float64).contiguous()
    poses = world_from_cam.reshape(-1, 8).to(torch.float64).contiguous()
    K = int(poses.shape[0])
    counts = torch.empty(max(K, 1), dtype=torch.int64, device=poses.device)
    cand = torch.empty(max(K, 1), dtype=torch.int32, device=poses.device)
    intr = np.ascontiguousarray(np.asarray(intrinsics, dtype=np.float64).reshape(6))
    ws = _lib.workspace(L.ec3r_local_candidates_workspace(K), poses.device, "local_cand")
    while True:
        amb = torch.empty((max(amb_cap, 1), 3), dtype=torch.int32, device=poses.device) if ambiguous else None
        n_amb = torch.zeros(1, dtype=torch.int64, device=poses.device) if ambiguous else None
        _lib.check(L.ec3r_local_candidates_ex(_lib.ptr(pts) if pts.shape[0] else None, int(pts.shape[0]),
                                              _lib.ptr(poses), K, intr.ctypes.data, float(tau_p), _lib.ptr(counts),
                                              _lib.ptr(cand), _lib.ptr(amb), int(amb_cap), _lib.ptr(n_amb),
                                              _lib.ptr(ws), ws.numel(), _lib.stream_ptr(stream)),
                   "ec3r_local_candidates_ex")
        if not ambiguous:
            return counts[:K], cand[:K]
        n = int(n_amb.item())
        if n <= amb_cap:
            return counts[:K], cand[:K], amb[:n].cpu().numpy()
        amb_cap = 2 * n


def _reference_visible(world_from_cam, k, positions: np.ndarray, idx: np.ndarray) -> np.ndarray:
    """Visibility of positions[idx] exactly as project_points computes it
    (geometry.py:87-109 under world_from_cam.inverse(), loops.py:129): the
    matmul runs over the whole array, as the reference's does."""
    pose = world_from_cam.inverse()
    pc = positions @ pose.rotation.matrix().T + pose.translation
    pc = pc[idx]
    z = pc[:, 2]
    safe_z = np.where(np.abs(z) > 1e-6, z, 1.0)
    u = k.fx * pc[:, 0] / safe_z + k.cx
    v = k.fy * pc[:, 1] / safe_z + k.cy
    return (z > 1e-6) & (u >= 0.0) & (u <= k.width - 1) & (v >= 0.0) & (v <= k.height - 1)


_local_guard_stats = {"ambiguous": 0, "flips": 0}


def detect_local_candidates(sparse_map, window, k, cfg) -> list:
    """loops.py:114-133 — keyframes of `window` ((kf_id, world_from_cam)
    pairs) that see more than cfg.tau_p of the live map's points.  Points
    within the margin band of the image border are re-decided on the host
    with the reference's expression (the device's summation order differs
    from BLAS's by ulps)."""
    from .types import sim3_to_vec

    _lib.lib()
    positions = sparse_map.positions()
    if len(positions) == 0 or len(window) == 0:
        return []
    pos = np.ascontiguousarray(np.asarray(positions, dtype=np.float64).reshape(-1, 3))
    pts = torch.as_tensor(pos, device="cuda")
    poses = torch.as_tensor(np.stack([sim3_to_vec(p) for _, p in window]), device="cuda")
    counts, cand, amb = local_candidates_device(pts, poses, (k.fx, k.fy, k.cx, k.cy, k.width, k.height),
                                                cfg.tau_p, ambiguous=True)
    c = cand.cpu().numpy().astype(bool)
    _local_guard_stats["ambiguous"] = int(len(amb))
    _local_guard_stats["flips"] = 0
    if len(amb):
        cnt = counts.cpu().numpy().astype(np.int64)
        for kk in np.unique(amb[:, 0]).tolist():
            rows = amb[amb[:, 0] == kk]
            vis = _reference_visible(window[kk][1], k, pos, rows[:, 1])
            delta = int(vis.sum()) - int(rows[:, 2].sum())
            if delta:
                _local_guard_stats["flips"] += int((vis != rows[:, 2].astype(bool)).sum())
                cnt[kk] += delta
                c[kk] = cnt[kk] / len(pos) > cfg.tau_p
    return [kf for (kf, _), ok in zip(window, c) if ok]


def last_local_guard_stats() -> dict:
    return dict(_local_guard_stats)


# -- loop verification (loops.py:136-153) on K5 + K9 -----------------------

try:  # pragma: no cover - exercised when the reference is installed
    from submap_slam.loops import APPEND, REJECT, REPLACE, LoopConfig, LoopVerdict
except ImportError:
    from dataclasses import dataclass, field

    from .types import RansacConfig

    REJECT, APPEND, REPLACE = "Reject", "AppendToBuffer", "ReplaceCurrent"  # loops.py:24-26

    @dataclass(frozen=True, eq=False)
    class LoopConfig:
        """loops.py:29-43."""

        tau1: float = 0.4
        tau2: float = 0.3
        tau_p: float = 0.7
        tau_global: float = 0.93
        tau_local: float = 0.96
        buffer_capacity: int = 5
        r_local: int = 3
        match_ratio: float = 0.8
        ransac: RansacConfig = field(default_factory=RansacConfig)

        def exclusion_zone(self) -> int:
            return 3 * self.buffer_capacity

    @dataclass
    class LoopVerdict:
        """loops.py:54-57."""

        verdict: str
        inlier_ratio: float


def verify_candidates(query_obs, candidate_obs, cfg) -> list:
    """verify_candidate (loops.py:136-153) for many candidates of one query:
    one matcher launch (K5, mutual NN + ratio test) over every (query,
    candidate) pair, then one batched homography RANSAC (K9) over the
    candidates with >= 4 matches; the tau_2 / tau_1 bands as the reference."""
    from .geometry import estimate_homography_ransac_batch
    from .tracking import match_batched

    cands = list(candidate_obs)
    if not cands:
        return []
    qd = np.asarray(query_obs.descriptors)
    live = [i for i, c in enumerate(cands) if len(qd) and len(c.descriptors)]
    pairs = match_batched([(qd, cands[i].descriptors) for i in live], cfg.match_ratio) if live else []
    probs, owners = [], []
    for i, m in zip(live, pairs):
        if len(m) >= 4:
            probs.append((np.asarray(query_obs.keypoints, float)[m[:, 0]],
                          np.asarray(cands[i].keypoints, float)[m[:, 1]]))
            owners.append(i)
    out = [LoopVerdict(REJECT, 0.0) for _ in cands]
    for i, res in zip(owners, estimate_homography_ransac_batch(probs, cfg.ransac)):
        r = res.inlier_ratio
        out[i] = LoopVerdict(REJECT if r <= cfg.tau2 else APPEND if r <= cfg.tau1 else REPLACE, r)
    return out


def verify_candidate(query_obs, candidate_obs, cfg):
    """loops.py:136-153 (one candidate)."""
    return verify_candidates(query_obs, [candidate_obs], cfg)[0]
