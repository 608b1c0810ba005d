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


# ---------------------------------------------------------------------------
# PnP RANSAC (geometry.py:414-474, called by tracking.py:208): the draws are
# the device replay of the reference's rng.choice stream (as above); each
# hypothesis is the reference's own host EPnP on its 4-point sample (its
# minimal poses depend on the exact null-space basis LAPACK returns,
# geometry.py:134-210, so they stay in the reference's host code); every
# hypothesis's reprojection pass over all correspondences runs on the device
# (ec3r_pnp_score, one warp per hypothesis), chunk by chunk, while the host
# walks the reference's acceptance rule and adaptive stop.  Decisions stay
# exact: a hypothesis with a point within 1e-9 (relative) of the pixel
# threshold, or a mean-error tie within 1e-9, is re-scored on the host with
# the reference expression.  The final all-inlier EPnP + Gauss-Newton refits
# are the reference's host code (:461-474).

_PNP_GUARD = 1e-9


def _ref_geometry():
    from .types import reference_module
    return reference_module("submap_slam.geometry")


def _pnp_problem(corrs, k):
    pts = np.array([c.point for c in corrs], dtype=float).reshape(-1, 3)
    pix = np.array([c.pixel for c in corrs], dtype=float).reshape(-1, 2)
    norm_pix = np.stack([(pix[:, 0] - k.cx) / k.fx, (pix[:, 1] - k.cy) / k.fy], axis=1)
    return pts, pix, norm_pix


def solve_pnp_ransac_batch(problems: Sequence, cfg: RansacConfig = RansacConfig(), seeds=None, chunk: int = 8,
                           stream=None, stats: Optional[dict] = None) -> list:
    """problems: sequence of (corrs, intrinsics).  One RansacResult per
    problem, or the exception instance the reference raises for it
    (TooFewCorrespondences, NoConsensus); equal to solve_pnp_ransac(corrs, k,
    cfg with seed=seeds[i])."""
    from .types import NoConsensus

    rg = _ref_geometry()
    L = _lib.lib()
    P = len(problems)
    if P == 0:
        return []
    seeds = [cfg.seed] * P if seeds is None else list(seeds)
    out: list = [None] * P
    data = []
    for p, (corrs, k) in enumerate(problems):
        n = len(corrs)
        if n < 4:
            out[p] = TooFewCorrespondences(f"PnP needs >= 4 correspondences, got {n}")
            data.append(None)
            continue
        data.append(_pnp_problem(corrs, k))
    live = [p for p in range(P) if data[p] is not None]
    if not live:
        return out
    iters = int(cfg.max_iterations)
    dev = torch.device("cuda", torch.cuda.current_device())
    h2d = lambda a: torch.as_tensor(np.ascontiguousarray(a)).to(dev)  # noqa: E731
    ns = np.array([len(data[p][0]) for p in live], np.int64)
    off_h = np.concatenate([[0], np.cumsum(ns)]).astype(np.int64)
    pts_d = h2d(np.concatenate([data[p][0] for p in live]))
    pix_d = h2d(np.concatenate([data[p][1] for p in live]))
    off_d = h2d(off_h)
    K4_d = h2d(np.array([[problems[p][1].fx, problems[p][1].fy, problems[p][1].cx, problems[p][1].cy]
                         for p in live], np.float64))
    state = h2d(np.stack([pcg_state(seeds[p]) for p in live]).view(np.int64))
    samples = torch.empty((len(live), max(iters, 1), 4), dtype=torch.int32, device=dev)
    st = _lib.stream_ptr(stream)
    ws = _lib.workspace(L.ec3r_ransac_draws_workspace(len(live)), dev, "pnp_draws")
    _lib.check(L.ec3r_ransac_draws(_lib.ptr(off_d), len(live), _lib.ptr(state), iters, _lib.ptr(samples),
                                   _lib.ptr(ws), ws.numel(), st), "ec3r_ransac_draws")
    samples_h = samples.cpu().numpy()
    thr = float(cfg.pixel_threshold)
    # per-problem walk state (geometry.py:431-455)
    S = [dict(it=0, max_iters=iters, best_count=0, best_err=np.inf, best_pose=None, exact_best=True)
         for _ in live]
    n_scored = n_rescored = 0
    width = max(1, int(chunk))
    while True:
        hyps, owner, poses = [], [], []
        for li, p in enumerate(live):
            s = S[li]
            if s["it"] >= s["max_iters"]:
                continue
            pts, pix, norm_pix = data[p]
            lo, hi = s["it"], min(s["max_iters"], s["it"] + width)
            for it in range(lo, hi):
                pose = rg._epnp(pts[samples_h[li, it]], norm_pix[samples_h[li, it]])
                poses.append((li, it, pose))
                if pose is not None:
                    R = pose.rotation.matrix()
                    hyps.append(np.concatenate([R.reshape(-1), pose.translation]))
                    owner.append(li)
        if not poses:
            break
        if hyps:
            H = len(hyps)
            hyp_d = h2d(np.asarray(hyps, np.float64))
            own_d = h2d(np.asarray(owner, np.int32))
            cnt_d = torch.empty(H, dtype=torch.int32, device=dev)
            sum_d = torch.empty(H, dtype=torch.float64, device=dev)
            amb_d = torch.empty(H, dtype=torch.int32, device=dev)
            _lib.check(L.ec3r_pnp_score(_lib.ptr(pts_d), _lib.ptr(pix_d), _lib.ptr(off_d), _lib.ptr(K4_d),
                                        _lib.ptr(hyp_d), _lib.ptr(own_d), H, thr, _PNP_GUARD, _lib.ptr(cnt_d),
                                        _lib.ptr(sum_d), _lib.ptr(amb_d), st), "ec3r_pnp_score")
            cnt_h, sum_h, amb_h = cnt_d.cpu().numpy(), sum_d.cpu().numpy(), amb_d.cpu().numpy()
            n_scored += H
        h = 0
        for li, it, pose in poses:  # chunks are in iteration order per problem
            s = S[li]
            if pose is None:
                if it < s["max_iters"]:
                    s["it"] = it + 1
                continue
            hi_ = h
            h += 1
            if it >= s["max_iters"]:  # past the adaptive stop: drawn but never reached
                continue
            s["it"] = it + 1
            p = live[li]
            pts, pix, _ = data[p]
            exact = bool(amb_h[hi_])
            count = int(cnt_h[hi_])
            mean_err = float(sum_h[hi_] / count) if count else np.inf
            if exact:  # the reference expression (geometry.py:442-445)
                err = rg._reprojection_errors(pose, problems[p][1], pts, pix)
                mask = err < thr
                count = int(mask.sum())
                mean_err = float(err[mask].mean()) if count else np.inf
                n_rescored += 1
            if count == s["best_count"] and count and (not exact or not s["exact_best"]) and \
                    abs(mean_err - s["best_err"]) <= _PNP_GUARD * max(abs(s["best_err"]), 1e-300):
                # mean-error tie within the device's rounding: decide on exact means
                err = rg._reprojection_errors(pose, problems[p][1], pts, pix)
                m = err < thr
                mean_err = float(err[m].mean())
                if not s["exact_best"]:
                    eb = rg._reprojection_errors(s["best_pose"], problems[p][1], pts, pix)
                    s["best_err"] = float(eb[eb < thr].mean())
                    s["exact_best"] = True
                exact = True
                n_rescored += 1
            if count > s["best_count"] or (count == s["best_count"] and mean_err < s["best_err"]):
                s["best_count"], s["best_err"], s["best_pose"], s["exact_best"] = count, mean_err, pose, exact
                if count > 4:
                    w = count / len(pts)
                    denom = math.log(max(1e-12, 1.0 - w ** 4))
                    if denom < 0:
                        needed = math.log(max(1e-300, 1.0 - cfg.confidence)) / denom
                        s["max_iters"] = min(cfg.max_iterations, max(it + 1, int(math.ceil(needed))))
        width = min(2 * width, 128)  # the adaptive stop usually lands early: grow the chunk gently
    for li, p in enumerate(live):
        s = S[li]
        pts, pix, norm_pix = data[p]
        k = problems[p][1]
        if s["best_pose"] is None or s["best_count"] < max(cfg.min_inliers, 4):
            out[p] = NoConsensus(f"best consensus {s['best_count']} below min_inliers {cfg.min_inliers}")
            continue
        # final model (geometry.py:459-474): the reference's host refits
        best_mask = rg._reprojection_errors(s["best_pose"], k, pts, pix) < thr
        idx = np.flatnonzero(best_mask)
        pose = rg._epnp(pts[idx], norm_pix[idx]) or s["best_pose"]
        pose = rg.refine_pose_gauss_newton(pose, k, pts[idx], pix[idx])
        mask = rg._reprojection_errors(pose, k, pts, pix) < thr
        if int(mask.sum()) >= max(cfg.min_inliers, 4):
            refined = rg.refine_pose_gauss_newton(pose, k, pts[mask], pix[mask])
            mask2 = rg._reprojection_errors(refined, k, pts, pix) < thr
            if mask2.sum() >= mask.sum():
                pose, mask = refined, mask2
        out[p] = RansacResult(pose, mask, float(mask.sum()) / len(pts))
    if stats is not None:
        stats.update(hypotheses_scored=n_scored, host_rescored=n_rescored)
    return out


def solve_pnp_ransac(corrs, k, cfg: RansacConfig = RansacConfig()) -> RansacResult:
    """geometry.py:414-474 with device hypothesis scoring (see above)."""
    r = solve_pnp_ransac_batch([(corrs, k)], cfg)[0]
    if isinstance(r, Exception):
        raise r
    return r
