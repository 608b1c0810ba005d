"""Voxel-hash fusion / downsampling restatement (TEST ORACLE ONLY).

The reference has NO voxel fusion: ``Mapping.fused_cloud`` concatenates the
world points of all submaps (mapping.py:332-338) and SPEC.md:611 lists dense
fusion as a non-goal.  This module declares the rule the CUDA fusion kernel
implements; only its two ingredients are pinned by the reference:

  * the transform  x_w = global_pose.apply(cloud.points)   mapping.py:56-57,
    Sim3Transform.apply / quat_rotate  liegroups.py:259-260, 90-95
    (pinned bit-exactly through the golden fused-cloud fixture), and
  * the key format  _pack(floor(x / cell))  _kernels/_numpy.py:50-55,81,87.

Declared rule (``fuse_points``):
  (i)   points = world points of every submap, concatenated (fused_cloud),
  (ii)  drop points with confidence <= 0,
  (iii) cell = floor(x / cell_size) (float64 division), key = _pack(cell);
        points whose cell leaves the 21-bit range [-2**20, 2**20) on any axis
        are dropped and counted (``_pack`` would alias them silently),
  (iv)  per key: wsum = sum conf, centroid = sum(conf * x) / wsum (float64),
        count = number of points,
  (v)   output sorted by key ascending.
Parity: keys and counts bit-exact, centroids within 1e-4 m, wsum within
1e-4 relative (the GPU accumulates in float32 relative to the voxel corner,
in arbitrary order).
"""

from __future__ import annotations

import numpy as np

from .ref_numpy import PACK_OFFSET, pack


def voxel_cells(x, cell_size):
    """floor(x / cell) as int64 (_kernels/_numpy.py:81,87)."""
    return np.floor(np.asarray(x, dtype=float) / cell_size).astype(np.int64)


def fuse_points(x, conf, cell_size):
    """Apply rules (ii)-(v).  Returns dict(keys, centroid, wsum, count,
    n_out_of_range, n_in)."""
    x = np.asarray(x, dtype=float).reshape(-1, 3)
    conf = np.asarray(conf, dtype=float).reshape(-1)
    live = conf > 0
    x = x[live]
    conf = conf[live]
    cells = voxel_cells(x, cell_size)
    ok = np.all((cells >= -PACK_OFFSET) & (cells < PACK_OFFSET), axis=1)
    n_oor = int((~ok).sum())
    x, conf, cells = x[ok], conf[ok], cells[ok]
    keys = pack(cells)
    order = np.argsort(keys, kind="stable")
    keys_s = keys[order]
    uniq, start, count = np.unique(keys_s, return_index=True, return_counts=True)
    wx = (x * conf[:, None])[order]
    wsum = np.add.reduceat(conf[order], start) if len(uniq) else np.zeros(0)
    sx = np.add.reduceat(wx, start, axis=0) if len(uniq) else np.zeros((0, 3))
    centroid = sx / wsum[:, None] if len(uniq) else np.zeros((0, 3))
    return dict(keys=uniq.astype(np.int64), centroid=centroid, wsum=wsum,
                count=count.astype(np.int64), n_out_of_range=n_oor, n_in=int(len(conf)))


def fuse_submaps(submaps, globals_, cell_size):
    """Rule (i) + fuse_points over dense submaps (see ref_numpy layout)."""
    from .ref_numpy import fused_cloud

    x, conf = fused_cloud(submaps, globals_)
    return fuse_points(x, conf, cell_size)


def fuse_submaps_streamed(submaps, globals_, cell_size, chunk=16):
    """fuse_submaps in bounded memory (TEST ORACLE ONLY): rules (i)-(v)
    applied to groups of ``chunk`` submaps, whose per-key partial sums
    (Σconf·x, Σconf, count) are merged by key.  Keys, counts and
    n_out_of_range are identical to fuse_submaps; the float64 sums differ
    only by summation order (far below the 1e-4 parity tolerances)."""
    from .ref_numpy import world_points

    parts = []
    n_oor = n_in = 0
    for g0 in range(0, len(submaps), chunk):
        xs, cs = [], []
        for sm, (s, q, t) in zip(submaps[g0:g0 + chunk], globals_[g0:g0 + chunk]):
            x, c = world_points(sm, s, q, t)
            xs.append(x)
            cs.append(c)
        f = fuse_points(np.concatenate(xs), np.concatenate(cs), cell_size)
        n_oor += f["n_out_of_range"]
        n_in += f["n_in"]
        parts.append((f["keys"], f["centroid"] * f["wsum"][:, None], f["wsum"], f["count"]))
    if not parts:
        return fuse_points(np.zeros((0, 3)), np.zeros(0), cell_size)
    keys = np.concatenate([p[0] for p in parts])
    order = np.argsort(keys, kind="stable")
    keys_s = keys[order]
    uniq, start = np.unique(keys_s, return_index=True)
    sx = np.add.reduceat(np.concatenate([p[1] for p in parts])[order], start, axis=0)
    wsum = np.add.reduceat(np.concatenate([p[2] for p in parts])[order], start)
    count = np.add.reduceat(np.concatenate([p[3] for p in parts])[order], start)
    return dict(keys=uniq.astype(np.int64), centroid=sx / wsum[:, None], wsum=wsum,
                count=count.astype(np.int64), n_out_of_range=n_oor, n_in=n_in)
