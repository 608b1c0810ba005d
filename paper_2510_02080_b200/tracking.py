"""Drop-in for the matcher of ``submap_slam.tracking`` (tracking.py:143-194):
brute-force mutual-NN + Lowe-ratio descriptor matching on the B200 path
(K5: tcgen05 similarity pass + certified float64 re-scoring, csrc/match_*.cu).

``match_descriptors`` / ``match_to_map`` keep the reference signatures and
return exactly the reference's matches; ``match_batched`` scores many frame
pairs (tracking frames, a local-loop window) in one launch.
"""

from __future__ import annotations

from typing import Optional, Sequence

import numpy as np
import torch

from . import _lib
from .types import Correspondence2D3D


def _pad_cols(t: torch.Tensor, D: int) -> torch.Tensor:
    if t.shape[1] == D:
        return t.contiguous()
    out = torch.zeros((t.shape[0], D), dtype=t.dtype, device=t.device)
    out[:, : t.shape[1]] = t
    return out


def padded_dim(d: int) -> int:
    return max(16, ((int(d) + 15) // 16) * 16)


def to_bf16_bits(x: torch.Tensor) -> torch.Tensor:
    """float tensor -> bf16 (round-to-nearest-even) raw bits as int16."""
    return x.to(torch.bfloat16).view(torch.int16)


def match_batched_device(A_bits: torch.Tensor, B_bits: torch.Tensor, A_x, B_x, exact_dtype: int,
                         a_off: np.ndarray, b_off: np.ndarray, ratio: float, norm_bound: float = 0.0, stream=None,
                         b_row: Optional[np.ndarray] = None):
    """One launch sequence of ec3r_match_batched.

    A_bits/B_bits: (rows, D) int16 bf16 bits (D % 16 == 0); A_x/B_x: exact
    rows (None when exact_dtype == 0, else float32/float64 (rows, D));
    a_off/b_off: host int64 (P+1) row offsets.  b_row (host int64 per pair,
    optional): pair p's map rows start at B row b_row[p] instead of
    b_off[p], so frames tracked against the same local map share its rows
    (ec3r_match_batched_rows).  Returns (match_b (sumN,) int32, n_match (P,)
    int32) CUDA tensors."""
    L = _lib.lib()
    P = len(a_off) - 1
    D = A_bits.shape[1]
    dev = A_bits.device
    a_off = np.ascontiguousarray(np.asarray(a_off, np.int64))
    b_off = np.ascontiguousarray(np.asarray(b_off, np.int64))
    ta, tb = int(a_off[-1]), int(b_off[-1])
    match_b = torch.empty(max(ta, 1), dtype=torch.int32, device=dev)
    n_match = torch.empty(max(P, 1), dtype=torch.int32, device=dev)
    ws_bytes = L.ec3r_match_workspace(a_off.ctypes.data, b_off.ctypes.data, P)
    ws = _lib.workspace(ws_bytes, dev, "match")
    if b_row is None:
        _lib.check(L.ec3r_match_batched(_lib.ptr(A_bits), _lib.ptr(B_bits), _lib.ptr(A_x), _lib.ptr(B_x),
                                        int(exact_dtype), a_off.ctypes.data, b_off.ctypes.data, P, D, float(ratio),
                                        float(norm_bound), _lib.ptr(match_b), _lib.ptr(n_match), _lib.ptr(ws),
                                        ws.numel(), _lib.stream_ptr(stream)), "ec3r_match_batched")
    else:
        b_row = np.ascontiguousarray(np.asarray(b_row, np.int64))
        _lib.check(L.ec3r_match_batched_rows(_lib.ptr(A_bits), _lib.ptr(B_bits), _lib.ptr(A_x), _lib.ptr(B_x),
                                             int(exact_dtype), a_off.ctypes.data, b_off.ctypes.data,
                                             b_row.ctypes.data, int(B_bits.shape[0]), P, D, float(ratio),
                                             float(norm_bound), _lib.ptr(match_b), _lib.ptr(n_match), _lib.ptr(ws),
                                             ws.numel(), _lib.stream_ptr(stream)), "ec3r_match_batched_rows")
    _last.update(ws=ws, ta=ta, tb=tb, P=P)
    return match_b[:ta], n_match[:P]


_last: dict = {}


def last_match_stats(stream=None) -> dict:
    """Rows / columns of the last match_batched_device call that needed the
    float64 full re-scan (the tensor-core pass certified the rest)."""
    import ctypes as C

    L = _lib.lib()
    r, c = C.c_int64(), C.c_int64()
    _lib.check(L.ec3r_match_stats(_lib.ptr(_last["ws"]), _last["ta"], _last["tb"], _last["P"], C.byref(r),
                                  C.byref(c), _lib.stream_ptr(stream)), "ec3r_match_stats")
    return {"rows_rescanned": r.value, "cols_rescanned": c.value, "rows": _last["ta"], "cols": _last["tb"]}


def prepare_rows(descs: Sequence, D: int):
    """Stack host descriptor arrays into device bf16 bits + exact rows.
    Returns (bits, exact, exact_dtype, offsets)."""
    arrs = [np.asarray(d, dtype=np.float64).reshape(len(d), -1) if len(d) else np.zeros((0, D)) for d in descs]
    off = np.zeros(len(arrs) + 1, np.int64)
    off[1:] = np.cumsum([len(a) for a in arrs])
    host = np.zeros((int(off[-1]), D))
    for a, o in zip(arrs, off[:-1]):
        host[o:o + len(a), : a.shape[1]] = a
    x = torch.as_tensor(host, device="cuda")
    bits = to_bf16_bits(x)
    exact_bf16 = bool(torch.equal(bits.view(torch.bfloat16).double(), x))
    if exact_bf16:
        return bits, None, 0, off
    return bits, x, 2, off


def match_batched(pairs: Sequence, ratio: float):
    """Many (desc_a, desc_b) frame pairs in one launch; returns a list of
    (K, 2) int64 arrays of (ia, ib) ascending in ia (match_descriptors
    semantics per pair)."""
    _lib.lib()
    if not pairs:
        return []
    dims = [np.asarray(a).shape[1] for a, b in pairs if len(a)] + [np.asarray(b).shape[1] for a, b in pairs if len(b)]
    D = padded_dim(max(dims) if dims else 16)
    A_bits, A_x, ta, a_off = prepare_rows([a for a, _ in pairs], D)
    B_bits, B_x, tb, b_off = prepare_rows([b for _, b in pairs], D)
    exact = 0 if (ta == 0 and tb == 0) else 2
    if exact == 2:
        A_x = A_bits.view(torch.bfloat16).double() if A_x is None else A_x
        B_x = B_bits.view(torch.bfloat16).double() if B_x is None else B_x
    mb, _ = match_batched_device(A_bits, B_bits, A_x, B_x, exact, a_off, b_off, ratio)
    mb = mb.cpu().numpy()
    out = []
    for p in range(len(pairs)):
        seg = mb[a_off[p]:a_off[p + 1]]
        ia = np.flatnonzero(seg >= 0)
        out.append(np.stack([ia, seg[ia].astype(np.int64)], axis=1).astype(np.int64))
    return out


def match_descriptors(desc_a, desc_b, ratio: float) -> list[tuple[int, int]]:
    """tracking.py:143-170 — mutual-NN matches (a_idx, b_idx) passing the
    ratio test (row side, as the reference implements it)."""
    if len(desc_a) == 0 or len(desc_b) == 0:
        return []
    (m,) = match_batched([(desc_a, desc_b)], ratio)
    return [(int(a), int(b)) for a, b in m]


def match_to_map(obs, sparse_map, cfg):
    """tracking.py:173-194 with the matcher on the B200 path."""
    pts = sparse_map.points()
    if not pts or len(obs.keypoints) == 0:
        return [], np.zeros(0, dtype=int), np.zeros(0, dtype=int)
    desc_map = np.array([p.descriptor for p in pts])
    pairs = match_descriptors(obs.descriptors, desc_map, cfg.ratio)
    corrs, obs_idx, point_ids = [], [], []
    for ia, ib in pairs:
        p = pts[ib]
        corrs.append(Correspondence2D3D(obs.keypoints[ia], p.position, p.id))
        obs_idx.append(ia)
        point_ids.append(p.id)
    return corrs, np.array(obs_idx, dtype=int), np.array(point_ids, dtype=int)
