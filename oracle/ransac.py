"""Restatement of the reference's homography RANSAC (TEST ORACLE ONLY).

estimate_homography_ransac (``geometry.py:594-640``) with its helpers
``_hartley_normalize`` (:534-543), ``_dlt_homography`` (:546-556),
``_symmetric_transfer_errors`` (:558-572) and ``_sample_degenerate``
(:575-583), restated for the checker of K9 (``csrc/ransac.cu``).  Pinned to
the reference through ``tests/golden/ransac.npz`` (``make_golden.gen_ransac``
runs the unmodified reference on its own test scenes and random mixtures).

``Pcg64Replay`` restates what K9 replays on the device: numpy's PCG64
(128-bit LCG, XSL-RR output, 32-bit halves buffered) and the path
``Generator.choice(n, 4, replace=False)`` takes (Floyd's sampling with
Lemire-bounded integers, then a Fisher-Yates shuffle of the four).  It is
pinned to ``rng.choice`` draws stored in the same fixture.
"""

from __future__ import annotations

import math

import numpy as np

_M64 = (1 << 64) - 1
_M128 = (1 << 128) - 1
_PCG_MULT = 0x2360ED051FC65DA44385DF649FCCF645


class Pcg64Replay:
    def __init__(self, seed):
        st = np.random.default_rng(seed).bit_generator.state
        self.s, self.inc = int(st["state"]["state"]), int(st["state"]["inc"])
        self.has32, self.u32 = int(st["has_uint32"]), int(st["uinteger"])

    def next64(self):
        self.s = (self.s * _PCG_MULT + self.inc) & _M128
        hi, lo = self.s >> 64, self.s & _M64
        rot = hi >> 58
        x = hi ^ lo
        return ((x >> rot) | (x << ((64 - rot) & 63))) & _M64

    def next32(self):
        if self.has32:
            self.has32 = 0
            return self.u32
        v = self.next64()
        self.has32, self.u32 = 1, v >> 32
        return v & 0xFFFFFFFF

    def bounded(self, r):
        """Uniform integer in [0, r], r < 2^32 (Lemire)."""
        if r == 0:
            return 0
        if r == 0xFFFFFFFF:
            return self.next32()
        ex = r + 1
        m = self.next32() * ex
        if (m & 0xFFFFFFFF) < ex:
            thr = (0xFFFFFFFF - r) % ex
            while (m & 0xFFFFFFFF) < thr:
                m = self.next32() * ex
        return m >> 32

    def choice4(self, n):
        idx = []
        for j in range(n - 4, n):
            v = self.bounded(j)
            idx.append(j if v in idx else v)
        for i in (3, 2, 1):
            k = self.bounded(i)
            idx[i], idx[k] = idx[k], idx[i]
        return idx


def hartley(pts):
    c = pts.mean(axis=0)
    d = np.linalg.norm(pts - c, axis=1).mean()
    d = 1.0 if d < 1e-12 else d
    s = math.sqrt(2.0) / d
    t = np.array([[s, 0.0, -s * c[0]], [0.0, s, -s * c[1]], [0.0, 0.0, 1.0]])
    return (np.concatenate([pts, np.ones((len(pts), 1))], axis=1) @ t.T)[:, :2], t


def dlt(src, dst):
    sn, ts = hartley(src)
    dn, td = hartley(dst)
    rows = []
    for (x, y), (u, v) in zip(sn, dn):
        rows.append([-x, -y, -1.0, 0.0, 0.0, 0.0, u * x, u * y, u])
        rows.append([0.0, 0.0, 0.0, -x, -y, -1.0, v * x, v * y, v])
    _, sv, vt = np.linalg.svd(np.array(rows))
    if len(src) > 4 and sv[-2] < 1e-12:
        return None
    h = vt[-1].reshape(3, 3)
    if abs(np.linalg.det(h)) < 1e-12:
        return None
    h = np.linalg.inv(td) @ h @ ts
    return h / h[2, 2] if abs(h[2, 2]) > 1e-12 else None


def transfer_errors(h, src, dst):
    def tr(m, p):
        ph = np.concatenate([p, np.ones((len(p), 1))], axis=1) @ m.T
        w = ph[:, 2]
        bad = np.abs(w) < 1e-12
        out = ph[:, :2] / np.where(bad, 1.0, w)[:, None]
        out[bad] = 1e9
        return out

    d1 = np.sum((tr(h, src) - dst) ** 2, axis=1)
    d2 = np.sum((tr(np.linalg.inv(h), dst) - src) ** 2, axis=1)
    return np.sqrt(0.5 * (d1 + d2))


def degenerate(p):
    for drop in range(4):
        a, b, c = np.delete(p, drop, axis=0)
        d1, d2 = b - a, c - a
        if abs(d1[0] * d2[1] - d1[1] * d2[0]) < 1e-9:
            return True
    return False


def hypotheses(src, dst, pixel_threshold, iters, seed):
    """Per-iteration inlier counts of the full budget (-1 = skipped), the
    quantity K9's score launch produces."""
    n = len(src)
    rng = np.random.default_rng(seed)
    out = np.full(iters, -1, np.int64)
    for it in range(iters):
        smp = rng.choice(n, size=4, replace=False)
        if degenerate(src[smp]) or degenerate(dst[smp]):
            continue
        h = dlt(src[smp], dst[smp])
        if h is not None:
            out[it] = int((transfer_errors(h, src, dst) < pixel_threshold).sum())
    return out


def estimate_homography_ransac(src, dst, pixel_threshold=2.0, confidence=0.999, max_iterations=1000, seed=0):
    """Returns (model 3x3, inlier mask, inlier ratio)."""
    src = np.asarray(src, float).reshape(-1, 2)
    dst = np.asarray(dst, float).reshape(-1, 2)
    n = len(src)
    if n < 4:
        raise ValueError("homography needs >= 4 pairs")
    rng = np.random.default_rng(seed)
    best_count, best_mask, best_h = 0, None, None
    limit, it = max_iterations, 0
    while it < limit:
        it += 1
        smp = rng.choice(n, size=4, replace=False)
        if degenerate(src[smp]) or degenerate(dst[smp]):
            continue
        h = dlt(src[smp], dst[smp])
        if h is None:
            continue
        mask = transfer_errors(h, src, dst) < pixel_threshold
        c = int(mask.sum())
        if c <= best_count:
            continue
        best_count, best_mask, best_h = c, mask, h
        if c > 4:
            denom = math.log(max(1e-12, 1.0 - (c / n) ** 4))
            if denom < 0:
                need = math.log(max(1e-300, 1.0 - confidence)) / denom
                limit = min(max_iterations, max(it, int(math.ceil(need))))
    if best_h is None:
        return np.eye(3), np.zeros(n, bool), 0.0
    if best_count >= 4:
        h = dlt(src[best_mask], dst[best_mask])
        if h is not None:
            mask = transfer_errors(h, src, dst) < pixel_threshold
            if mask.sum() >= best_count:
                best_h, best_mask, best_count = h, mask, int(mask.sum())
    return best_h, best_mask, best_count / n
