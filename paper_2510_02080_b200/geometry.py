"""Drop-in for the reference's homography RANSAC (``geometry.py:594-640``),
batched: K9 (``csrc/ransac.cu``) scores every hypothesis of every problem's
``max_iterations`` budget in one pass on the B200, replaying the reference's
``np.random.default_rng(cfg.seed)`` draws bit-for-bit; the host then walks the
per-iteration inlier counts with the reference's acceptance rule and adaptive
stop (Python floats, ``math.log``, as in ``:620-625``), and one more launch
computes the chosen model's mask, the all-inlier refit and the keep rule
(``:633-639``).

``estimate_homography_ransac(matches, cfg)`` keeps the reference signature;
``estimate_homography_ransac_batch`` takes many match sets (one per loop
candidate, ``loops.verify_candidate``) and returns one ``RansacResult`` each.
There is no CPU fallback.
"""

from __future__ import annotations

import functools
import math
from typing import Optional, Sequence

import numpy as np
import torch

from . import _lib
from .types import RansacConfig, RansacResult, TooFewCorrespondences


@functools.lru_cache(maxsize=4096)
def _pcg_state_cached(seed: int) -> tuple:
    return tuple(int(x) for x in _pcg_state(seed))


def pcg_state(seed) -> np.ndarray:
    """numpy PCG64 state of default_rng(seed) as 6 uint64 (state hi/lo, inc
    hi/lo, has_uint32, uinteger) — the stream K9 replays.  Integer seeds are
    cached (SeedSequence hashing costs ~20 us per generator)."""
    if isinstance(seed, (int, np.integer)):
        return np.array(_pcg_state_cached(int(seed)), np.uint64)
    return _pcg_state(seed)


def _pcg_state(seed) -> np.ndarray:
    st = np.random.default_rng(seed).bit_generator.state
    s, inc = int(st["state"]["state"]), int(st["state"]["inc"])
    m = (1 << 64) - 1
    return np.array([s >> 64, s & m, inc >> 64, inc & m, int(st["has_uint32"]), int(st["uinteger"])], np.uint64)


def _walk(improvements, counts_row, n: int, cfg: RansacConfig) -> int:
    best_i, max_iters = -1, int(cfg.max_iterations)
    for i in improvements:
        it = int(i) + 1
        if it > max_iters:
            break
        c = int(counts_row[i])
        best_i = int(i)
        if c > 4:
            w = c / n
            denom = math.log(max(1e-12, 1.0 - w ** 4))
            if denom < 0:
                needed = math.log(max(1e-300, 1.0 - cfg.confidence)) / denom
                max_iters = min(cfg.max_iterations, max(it, int(math.ceil(needed))))
    return best_i


def _improvements(counts: np.ndarray) -> np.ndarray:
    """Mask of iterations whose count beats every earlier one (and 0): the
    only places the reference's loop changes state."""
    c = np.maximum(counts, 0)
    prev = np.zeros_like(c)
    prev[..., 1:] = np.maximum.accumulate(c, axis=-1)[..., :-1]
    return counts > prev


def walk_counts(counts: np.ndarray, n: int, cfg: RansacConfig) -> int:
    """The reference's sequential RANSAC loop (geometry.py:607-625) over the
    per-iteration inlier counts (-1 = skipped).  Returns the 0-based
    iteration whose hypothesis wins, or -1."""
    counts = np.asarray(counts)
    return _walk(np.flatnonzero(_improvements(counts)), counts, n, cfg)


def walk_counts_batch(counts: np.ndarray, ns, cfg: RansacConfig) -> np.ndarray:
    """walk_counts for every row of a (P, iters) count matrix."""
    rows, cols = np.nonzero(_improvements(counts))
    starts = np.searchsorted(rows, np.arange(len(ns) + 1))
    return np.array([_walk(cols[starts[p]:starts[p + 1]], counts[p], int(ns[p]), cfg) for p in range(len(ns))],
                    np.int32)


def estimate_homography_ransac_batch(problems: Sequence, cfg: RansacConfig = RansacConfig(),
                                     seeds: Optional[Sequence[int]] = None, stream=None,
                                     return_samples: bool = False):
    """problems: sequence of (src (n, 2), dst (n, 2)) pixel arrays (or match
    lists as the reference takes).  One RansacResult per problem, equal to
    estimate_homography_ransac(matches, cfg with seed=seeds[i])."""
    L = _lib.lib()
    srcs, dsts = [], []
    for pr in problems:
        if isinstance(pr, (list, tuple)) and len(pr) == 2 and not np.isscalar(pr[0]) and np.ndim(pr[0]) == 2:
            s, d = pr
        else:  # list of (src_pt, dst_pt) as the reference takes
            s = np.array([m[0] for m in pr], dtype=float).reshape(-1, 2)
            d = np.array([m[1] for m in pr], dtype=float).reshape(-1, 2)
        s = np.asarray(s, np.float64).reshape(-1, 2)
        d = np.asarray(d, np.float64).reshape(-1, 2)
        if len(s) < 4:
            raise TooFewCorrespondences(f"homography needs >= 4 pairs, got {len(s)}")
        srcs.append(s)
        dsts.append(d)
    P = len(srcs)
    if P == 0:
        return []
    seeds = [cfg.seed] * P if seeds is None else list(seeds)
    iters = int(cfg.max_iterations)
    ns = np.array([len(s) for s in srcs], np.int64)
    off_h = np.concatenate([[0], np.cumsum(ns)]).astype(np.int64)
    dev = torch.device("cuda", torch.cuda.current_device())
    h2d = lambda a: torch.as_tensor(np.ascontiguousarray(a)).to(dev, non_blocking=False)  # noqa: E731
    src = h2d(np.concatenate(srcs))
    dst = h2d(np.concatenate(dsts))
    off = h2d(off_h)
    state = h2d(np.stack([pcg_state(s) for s in seeds]).view(np.int64))
    counts = torch.empty((P, max(iters, 1)), dtype=torch.int32, device=dev)
    samples = torch.empty((P, max(iters, 1), 4), dtype=torch.int32, device=dev) if return_samples else None
    ws = _lib.workspace(L.ec3r_homography_workspace(P, iters), dev, "ransac")
    st = _lib.stream_ptr(stream)
    _lib.check(L.ec3r_homography_ransac_score(_lib.ptr(src), _lib.ptr(dst), _lib.ptr(off), P, _lib.ptr(state), iters,
                                              float(cfg.pixel_threshold), _lib.ptr(counts), _lib.ptr(samples),
                                              _lib.ptr(ws), ws.numel(), st), "ec3r_homography_ransac_score")
    counts_h = counts.cpu().numpy()
    best = walk_counts_batch(counts_h[:, :iters], ns, cfg)
    best_d = h2d(best)
    model = torch.empty((P, 9), dtype=torch.float64, device=dev)
    mask = torch.empty(int(off_h[-1]), dtype=torch.uint8, device=dev)
    cnt = torch.empty(P, dtype=torch.int32, device=dev)
    _lib.check(L.ec3r_homography_ransac_refit(_lib.ptr(src), _lib.ptr(dst), _lib.ptr(off), P, _lib.ptr(best_d), iters,
                                              float(cfg.pixel_threshold), _lib.ptr(model), _lib.ptr(mask),
                                              _lib.ptr(cnt), _lib.ptr(ws), ws.numel(), st),
               "ec3r_homography_ransac_refit")
    model_h, mask_h, cnt_h = model.cpu().numpy(), mask.cpu().numpy().astype(bool), cnt.cpu().numpy()
    out = []
    for p in range(P):
        n = int(ns[p])
        out.append(RansacResult(model_h[p].reshape(3, 3).copy(), mask_h[off_h[p]:off_h[p + 1]].copy(),
                                int(cnt_h[p]) / n))
    if return_samples:
        return out, counts_h, samples.cpu().numpy()
    return out


def estimate_homography_ransac(matches, cfg: RansacConfig = RansacConfig()) -> RansacResult:
    """geometry.py:594-640 on the B200 (see module doc)."""
    return estimate_homography_ransac_batch([matches], cfg)[0]
