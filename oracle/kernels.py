"""Restatement of the reference's native-kernel plugin slot (TEST ORACLE ONLY).

``submap_slam._kernels`` (``_kernels/__init__.py:12-33``) exports ``raycast``,
``nn_query`` and ``nn_dists`` with numpy-in / numpy-out semantics defined by
``_kernels/_numpy.py``.  This module restates those semantics per query / per
ray (plain loops over the shells, not the reference's vectorised layout) so
that the CUDA path (``paper_2510_02080_b200.kernels``) has a checker.  It is
pinned to the reference through ``tests/golden/kernels.npz``
(``tests/golden/make_golden.py`` runs the unmodified ``_numpy`` module).

nn_query (``_numpy.py:66-132``):
  * reference cells = floor(ref / cell) (float64), keys = _pack(cells)
    (``:50-55``); reference points are visited in key order, equal keys in
    original order (stable argsort, ``:82-84``);
  * per query, rings r = 0.._BRUTE_RING (8) of Chebyshev shells around the
    query cell, shells enumerated in meshgrid "ij" order (``:58-62``); every
    point of every shell cell is a candidate, in that order; the ring's best
    is its first minimum (stable lexsort, ``:108-113``), and it replaces the
    running best only when strictly smaller (``:117-120``);
  * the query is done once best <= r * cell (``:121-122``);
  * queries still open after ring 8 take the brute-force first minimum over
    all reference points in original order (``:126-131``);
  * distances are sqrt(dx^2 + dy^2 + dz^2) in float64, ref - query
    (``:105-106``); empty ref -> (inf, -1); empty query -> empty arrays.
raycast (``_numpy.py:29-47``, slab test ``:14-26``):
  * first-hit parameter over the room shell and the solid boxes, t = near
    when near > 1e-9 else far, a hit needs near <= far and far > 1e-9;
    rays parallel to a slab axis use the inside / outside rule; 0 where
    nothing is hit.
"""

from __future__ import annotations

import numpy as np

from .ref_numpy import PACK_OFFSET

EPS = 1e-9
BRUTE_RING = 8


def pack_cells(c):
    """_pack (_numpy.py:50-55) in wrapping int64 arithmetic."""
    c = np.asarray(c, dtype=np.int64)
    with np.errstate(over="ignore"):
        return (((c[..., 0] + PACK_OFFSET) << 42) | ((c[..., 1] + PACK_OFFSET) << 21) | (c[..., 2] + PACK_OFFSET))


def shell(r):
    """Chebyshev shell r in meshgrid 'ij' order (last axis fastest)."""
    out = []
    for i in range(-r, r + 1):
        for j in range(-r, r + 1):
            for k in range(-r, r + 1):
                if max(abs(i), abs(j), abs(k)) == r:
                    out.append((i, j, k))
    return np.array(out, dtype=np.int64).reshape(-1, 3)


def _dist(p, q):
    d = p - q
    return np.sqrt(d[..., 0] * d[..., 0] + d[..., 1] * d[..., 1] + d[..., 2] * d[..., 2])


def nn_query(query, ref, cell_size):
    query = np.asarray(query, dtype=float).reshape(-1, 3)
    ref = np.asarray(ref, dtype=float).reshape(-1, 3)
    nq = len(query)
    if nq == 0:
        return np.zeros(0), np.zeros(0, dtype=np.int64)
    if len(ref) == 0:
        return np.full(nq, np.inf), np.full(nq, -1, dtype=np.int64)
    keys = pack_cells(np.floor(ref / cell_size).astype(np.int64))
    order = np.argsort(keys, kind="stable")
    skeys = keys[order]
    sref = ref[order]
    # cell key -> [start, end) in the sorted arrays
    uk, starts, counts = np.unique(skeys, return_index=True, return_counts=True)
    table = {int(k): (int(s), int(s + n)) for k, s, n in zip(uk, starts, counts)}
    shells = [shell(r) for r in range(BRUTE_RING + 1)]
    qcells = np.floor(query / cell_size).astype(np.int64)
    best = np.full(nq, np.inf)
    out = np.full(nq, -1, dtype=np.int64)
    for i in range(nq):
        b, bi = np.inf, -1
        done = False
        for r in range(BRUTE_RING + 1):
            ck = pack_cells(qcells[i][None, :] + shells[r])
            rb, rbi = np.inf, -1
            for k in ck:
                span = table.get(int(k))
                if span is None:
                    continue
                d = _dist(sref[span[0]:span[1]], query[i])
                j = int(np.argmin(d))
                if d[j] < rb:  # first minimum in candidate order
                    rb, rbi = float(d[j]), span[0] + j
            if rb < b:
                b, bi = rb, rbi
            if b <= r * cell_size:
                done = True
                break
        if done:
            best[i], out[i] = b, int(order[bi])
        else:  # stray query: brute force, first minimum in original order
            d = _dist(ref, query[i])
            j = int(np.argmin(d))
            best[i], out[i] = float(d[j]), j
    return best, out


def nn_dists(query, ref, cell_size):
    return nn_query(query, ref, cell_size)[0]


def _slab(o, d, bmin, bmax):
    near, far = -np.inf, np.inf
    for a in range(3):
        if d[a] == 0.0:
            inside = bmin[a] <= o[a] <= bmax[a]
            t1, t2 = (-np.inf, np.inf) if inside else (np.inf, -np.inf)
        else:
            inv = 1.0 / d[a]
            t1 = (bmin[a] - o[a]) * inv
            t2 = (bmax[a] - o[a]) * inv
        near = max(near, min(t1, t2))
        far = min(far, max(t1, t2))
    return near, far


def raycast(origins, dirs, room_min, room_max, boxes):
    origins = np.asarray(origins, dtype=float).reshape(-1, 3)
    dirs = np.asarray(dirs, dtype=float).reshape(-1, 3)
    solids = [(np.asarray(room_min, float), np.asarray(room_max, float))] + \
        [(np.asarray(a, float), np.asarray(b, float)) for a, b in boxes]
    out = np.zeros(len(origins))
    for i in range(len(origins)):
        best = np.inf
        for bmin, bmax in solids:
            near, far = _slab(origins[i], dirs[i], bmin, bmax)
            if near <= far and far > EPS:
                best = min(best, near if near > EPS else far)
        out[i] = best if np.isfinite(best) else 0.0
    return out
