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
