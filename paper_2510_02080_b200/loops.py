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
                             device="cuda")
    kfs = np.asarray(order, dtype=np.int64)
    cp, cs, qp, qs, ep, es = retrieval_device(pooled, int(stride), int(cfg.exclusion_zone()),
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
        self.n = 0

    def append(self, kf_ids, pooled):
        pooled = torch.as_tensor(np.asarray(pooled, np.float64).reshape(-1, self.dim), device=self.device)
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
        self.vec[self.n:self.n + k] = pooled
        self.kf[self.n:self.n + k] = np.asarray(kf_ids, np.int64)
        self.n += k

    def score(self, stride: int, exclusion: int, tau_g: float, tau_l: float, k_begin: int = 0, k_end: int = -1):
        return retrieval_device(self.vec[: self.n], stride, exclusion, tau_g, tau_l, k_begin, k_end)

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
                            stream=None):
    """Projection counts of the map points (N, 3) float64 into K keyframes
    (world_from_cam: (K, 8) float64 {s, q, t}) in one launch.  Returns
    (counts (K,) int64, candidate (K,) int32) CUDA tensors; intrinsics =
    (fx, fy, cx, cy, width, height)."""
    L = _lib.lib()
    pts = positions.reshape(-1, 3).to(torch.float64).contiguous()
    poses = world_from_cam.reshape(-1, 8).to(torch.float64).contiguous()
    K = int(poses.shape[0])
    counts = torch.empty(max(K, 1), dtype=torch.int64, device=poses.device)
    cand = torch.empty(max(K, 1), dtype=torch.int32, device=poses.device)
    intr = np.ascontiguousarray(np.asarray(intrinsics, dtype=np.float64).reshape(6))
    ws = _lib.workspace(L.ec3r_local_candidates_workspace(K), poses.device, "local_cand")
    _lib.check(L.ec3r_local_candidates(_lib.ptr(pts) if pts.shape[0] else None, int(pts.shape[0]), _lib.ptr(poses),
                                       K, intr.ctypes.data, float(tau_p), _lib.ptr(counts), _lib.ptr(cand),
                                       _lib.ptr(ws), ws.numel(), _lib.stream_ptr(stream)), "ec3r_local_candidates")
    return counts[:K], cand[:K]


def detect_local_candidates(sparse_map, window, k, cfg) -> list:
    """loops.py:114-133 — keyframes of `window` ((kf_id, world_from_cam)
    pairs) that see more than cfg.tau_p of the live map's points."""
    from .types import sim3_to_vec

    _lib.lib()
    positions = sparse_map.positions()
    if len(positions) == 0 or len(window) == 0:
        return []
    pts = torch.as_tensor(np.ascontiguousarray(np.asarray(positions, dtype=np.float64)), device="cuda")
    poses = torch.as_tensor(np.stack([sim3_to_vec(p) for _, p in window]), device="cuda")
    _, cand = local_candidates_device(pts, poses, (k.fx, k.fy, k.cx, k.cy, k.width, k.height), cfg.tau_p)
    c = cand.cpu().numpy()
    return [kf for (kf, _), ok in zip(window, c) if ok]


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
