"""Drop-in for ``submap_slam.registration`` (registration.py:1-112) on the
B200 path: weighted Umeyama Sim(3) runs in the K2+K3 cluster kernel
(csrc/umeyama.cu) through ``ec3r_umeyama_batched``.

Same names, argument meaning, return values and exception precedence as the
reference: TooFewCorrespondences (n < 3) -> ValueError (shape) ->
AllZeroConfidence (sum w <= 0) -> DegenerateConfiguration (collinear source
or non-positive scale).
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np
import torch

from . import _lib
from .types import (AllZeroConfidence, DegenerateConfiguration, Sim3Transform,
                    TooFewCorrespondences, vec_to_sim3)


@dataclass(frozen=True, eq=False)
class Correspondence3D3D:
    """registration.py:19-25."""

    p: np.ndarray
    q: np.ndarray
    weight: float = 1.0


def normalize_confidences(confidences: Sequence[float]) -> np.ndarray:
    """registration.py:28-35 (host utility, no device work)."""
    c = np.asarray(confidences, dtype=float)
    if c.size == 0 or not np.any(c > 0):
        raise AllZeroConfidence("need at least one strictly positive confidence")
    if np.any(c < 0):
        raise ValueError("confidences must be non-negative")
    return c / c.sum()


def _dev(x, dtype=torch.float64) -> torch.Tensor:
    if isinstance(x, torch.Tensor):
        t = x.to(device="cuda", dtype=dtype)
    else:
        t = torch.as_tensor(np.ascontiguousarray(np.asarray(x, dtype=np.float64)), device="cuda")
        t = t.to(dtype)
    return t.contiguous()


def raise_for_status(status: int, n: int = 0) -> None:
    """Map an EC3R_ST_* code to the reference exception (registration.py:59-93)."""
    if status == _lib.ST_OK or status == _lib.ST_SKIP:
        return
    if status == _lib.ST_TOO_FEW:
        raise TooFewCorrespondences(f"need >= 3 correspondences, got {n}")
    if status == _lib.ST_ALL_ZERO:
        raise AllZeroConfidence("total weight must be positive")
    if status == _lib.ST_DEGENERATE:
        raise DegenerateConfiguration("source points are collinear or coincident")
    if status == _lib.ST_NONPOS_SCALE:
        raise DegenerateConfiguration("non-positive scale from degenerate input")
    raise RuntimeError(f"unknown registration status {status}")


def align_batched_device(p: torch.Tensor, q: torch.Tensor, w: Optional[torch.Tensor], offsets: torch.Tensor,
                         with_scale: bool = True, stream=None):
    """Batched Umeyama on device tensors.

    p, q: (sum n_b, 3) float64 CUDA; w: (sum n_b,) float64 or None;
    offsets: (B+1,) int64 CUDA.  Returns device tensors (sim3 (B,8), rms (B,),
    status (B,) int32) without synchronizing."""
    L = _lib.lib()
    B = offsets.numel() - 1
    sim3 = torch.empty((B, 8), dtype=torch.float64, device=p.device)
    rms = torch.empty(B, dtype=torch.float64, device=p.device)
    status = torch.empty(B, dtype=torch.int32, device=p.device)
    _lib.check(L.ec3r_umeyama_batched(_lib.ptr(p), _lib.ptr(q), _lib.ptr(w), _lib.ptr(offsets), B,
                                      int(bool(with_scale)), _lib.ptr(sim3), _lib.ptr(rms), _lib.ptr(status),
                                      None, 0, _lib.stream_ptr(stream)), "ec3r_umeyama_batched")
    return sim3, rms, status


def align_point_sets_batched(problems, with_scale: bool = True):
    """Many independent align_point_sets problems in ONE launch.

    problems: sequence of (p, q, weights-or-None).  Returns a list of
    (Sim3Transform or None, rms or None, exception or None) in input order."""
    _lib.lib()
    ps, qs, ws, offs, bad = [], [], [], [0], {}
    any_w = any(w is not None for _, _, w in problems)
    for i, (p, q, w) in enumerate(problems):
        p = np.asarray(p, dtype=float)
        q = np.asarray(q, dtype=float)
        n = p.shape[0]
        if n < 3:
            bad[i] = TooFewCorrespondences(f"need >= 3 correspondences, got {n}")
        elif q.shape != p.shape:
            bad[i] = ValueError("point sets must have matching shapes")
        if i in bad:
            p = np.zeros((0, 3))
            q = np.zeros((0, 3))
            w = None
        ps.append(p.reshape(-1, 3))
        qs.append(q.reshape(-1, 3))
        ws.append(np.ones(len(p)) if w is None else np.asarray(w, dtype=float).reshape(-1))
        offs.append(offs[-1] + len(p))
    if len(bad) < len(problems):
        P = _dev(np.concatenate(ps))
        Q = _dev(np.concatenate(qs))
        Wt = _dev(np.concatenate(ws)) if any_w else None
        O = torch.as_tensor(np.asarray(offs, np.int64), device="cuda")
        sim3, rms, status = align_batched_device(P, Q, Wt, O, with_scale)
        sim3, rms, status = sim3.cpu().numpy(), rms.cpu().numpy(), status.cpu().numpy()
    out = []
    for i in range(len(problems)):
        if i in bad:
            out.append((None, None, bad[i]))
            continue
        try:
            raise_for_status(int(status[i]), offs[i + 1] - offs[i])
            out.append((vec_to_sim3(sim3[i]), float(rms[i]), None))
        except (TooFewCorrespondences, AllZeroConfidence, DegenerateConfiguration) as e:
            out.append((None, None, e))
    return out


def align_point_sets(p, q, weights=None, with_scale: bool = True) -> tuple[Sim3Transform, float]:
    """registration.py:38-102 — weighted Umeyama alignment of q ~ s R p + t.

    Returns (transform, residual_rms); raises the reference's exceptions."""
    if isinstance(p, torch.Tensor) and p.is_cuda:
        n = p.shape[0]
        if n < 3:
            raise TooFewCorrespondences(f"need >= 3 correspondences, got {n}")
        if tuple(q.shape) != tuple(p.shape):
            raise ValueError("point sets must have matching shapes")
        w = None if weights is None else _dev(weights).reshape(-1)
        O = torch.tensor([0, n], dtype=torch.int64, device=p.device)
        sim3, rms, status = align_batched_device(_dev(p), _dev(q), w, O, with_scale)
        st = int(status.item())
        raise_for_status(st, n)
        return vec_to_sim3(sim3[0].cpu().numpy()), float(rms.item())
    ((t, r, e),) = align_point_sets_batched([(p, q, weights)], with_scale)
    if e is not None:
        raise e
    return t, r


def weighted_umeyama(corrs: Sequence[Correspondence3D3D]) -> tuple[Sim3Transform, float]:
    """registration.py:105-112."""
    if len(corrs) < 3:
        raise TooFewCorrespondences(f"need >= 3 correspondences, got {len(corrs)}")
    p = np.array([c.p for c in corrs], dtype=float)
    q = np.array([c.q for c in corrs], dtype=float)
    w = np.array([c.weight for c in corrs], dtype=float)
    return align_point_sets(p, q, w)
