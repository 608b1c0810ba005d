"""Local loop candidate detection restated (TEST ORACLE ONLY).

detect_local_candidates (loops.py:114-133): for each window keyframe
(kf_id, world_from_cam), project the live map's points with
project_points(world_from_cam.inverse(), K, positions) (geometry.py:87-109)
and keep the keyframe when visible.sum() / len(positions) > tau_p.  Pose
inverse: liegroups.py:217-219 (rinv = conj(q), t' = -rinv.apply(t)); the
rotation matrix is quat_to_matrix (liegroups.py:56-65).  Pinned to the
reference through tests/golden/local.npz.
"""

from __future__ import annotations

import numpy as np

Z_MIN = 1e-6  # geometry.py:23


def _quat_matrix(q):
    w, x, y, z = q
    return np.array([[1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)],
                     [2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)],
                     [2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)]])


def _rotate(q, p):
    v = np.asarray(q[1:], float)
    uv = 2.0 * np.cross(v, p)
    return p + q[0] * uv + np.cross(v, uv)


def visible_counts(positions, poses8, intr):
    """Per keyframe: number of points visible from world_from_cam.inverse()."""
    pts = np.asarray(positions, float).reshape(-1, 3)
    fx, fy, cx, cy, w, h = intr
    out = []
    for p8 in np.asarray(poses8, float).reshape(-1, 8):
        qi = np.array([p8[1], -p8[2], -p8[3], -p8[4]])
        ti = -_rotate(qi, p8[5:8])
        pc = pts @ _quat_matrix(qi).T + ti
        z = pc[:, 2]
        sz = np.where(np.abs(z) > Z_MIN, z, 1.0)
        u = fx * pc[:, 0] / sz + cx
        v = fy * pc[:, 1] / sz + cy
        vis = (z > Z_MIN) & (u >= 0.0) & (u <= w - 1) & (v >= 0.0) & (v <= h - 1)
        out.append(int(vis.sum()))
    return np.array(out, dtype=np.int64)


def local_candidates(positions, kf_ids, poses8, intr, tau_p):
    n = len(np.asarray(positions).reshape(-1, 3))
    if n == 0:
        return []
    c = visible_counts(positions, poses8, intr)
    return [int(k) for k, ci in zip(kf_ids, c) if ci / n > tau_p]
