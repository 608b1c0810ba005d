"""Numpy restatement of the reference hot-path functions (TEST ORACLE ONLY).

Every function follows the reference line by line, in float64, with the same
operation order where bit-exactness matters (keys, masks, matches).  File
citations are into ``/root/reference/pkg/src/submap_slam``.

Data layout used by the oracle and by the CUDA path alike (the "dense
submap" form of ``ReconstructionOutput``, backend.py:51-58):
  depth   (F, H, W) float, 0 where no surface
  conf    (F, H, W) float in [0, 1]
  frame_ids (F,) int
  pose_q  (F, 4) float64 unit quaternions (w, x, y, z), anchor_from_cam
  pose_t  (F, 3) float64
  K       (fx, fy, cx, cy)
Status strings stand in for the reference exception types so the oracle has
no dependency on the reference package (errors.py:12-53).
"""

from __future__ import annotations

import math

import numpy as np

STATUS_OK = "ok"
STATUS_TOO_FEW = "too_few"          # TooFewCorrespondences  registration.py:59-60
STATUS_SHAPE = "shape"              # ValueError             registration.py:61-62
STATUS_ALL_ZERO = "all_zero"        # AllZeroConfidence      registration.py:68-69
STATUS_DEGENERATE = "degenerate"    # DegenerateConfiguration registration.py:82-83,92-93
STATUS_SKIP = "skip"                # edge gated out (< min_correspondences) mapping.py:174,178

PACK_OFFSET = 1 << 20               # _kernels/_numpy.py:47


# --------------------------------------------------------------------------
# Lie-group value arithmetic (liegroups.py)

def quat_rotate(q, pts):
    """liegroups.py:90-95 — uv = 2 v x p;  p + w uv + v x uv."""
    q = np.asarray(q, dtype=float)
    w = q[0]
    v = q[1:]
    uv = 2.0 * np.cross(v, pts)
    return pts + w * uv + np.cross(v, uv)


def pose_apply(q, t, pts):
    """Pose3.apply, liegroups.py:208-209 (rotation.apply + translation)."""
    return quat_rotate(q, np.asarray(pts, dtype=float)) + np.asarray(t, dtype=float)


def sim3_apply(s, q, t, pts):
    """Sim3Transform.apply, liegroups.py:259-260."""
    return s * quat_rotate(q, np.asarray(pts, dtype=float)) + np.asarray(t, dtype=float)


def normalize_quat(q):
    """Rotation3.__post_init__, liegroups.py:139-142."""
    q = np.asarray(q, dtype=float)
    return q / np.linalg.norm(q)


def quat_to_matrix(q):
    """liegroups.py:55-64."""
    w, x, y, z = q
    return np.array(
        [
            [1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)],
            [2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)],
            [2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)],
        ]
    )


def matrix_to_quat(m):
    """Shepperd's method, liegroups.py:68-87."""
    t = np.trace(m)
    if t > 0:
        r = math.sqrt(1.0 + t)
        s = 0.5 / r
        q = np.array([0.5 * r, (m[2, 1] - m[1, 2]) * s, (m[0, 2] - m[2, 0]) * s,
                      (m[1, 0] - m[0, 1]) * s])
    else:
        i = int(np.argmax(np.diag(m)))
        j, k = (i + 1) % 3, (i + 2) % 3
        r = math.sqrt(1.0 + m[i, i] - m[j, j] - m[k, k])
        s = 0.5 / r
        q = np.empty(4)
        q[0] = (m[k, j] - m[j, k]) * s
        q[1 + i] = 0.5 * r
        q[1 + j] = (m[j, i] + m[i, j]) * s
        q[1 + k] = (m[k, i] + m[i, k]) * s
    return q / np.linalg.norm(q)


def canonical_quat(q):
    """q and -q are the same rotation (liegroups.py:175-178); pick w >= 0."""
    q = np.asarray(q, dtype=float)
    if q[0] < 0 or (q[0] == 0 and next((c for c in q[1:] if c != 0), 0) < 0):
        return -q
    return q


def sim3_compose(a, b):
    """sim3_compose, liegroups.py:275-281; a, b = (s, q, t)."""
    sa, qa, ta = a
    sb, qb, tb = b
    return (sa * sb, normalize_quat(quat_mul(qa, qb)), sa * quat_rotate(qa, tb) + ta)


def quat_mul(a, b):
    """Hamilton product (w, x, y, z) — liegroups.py quat_mul."""
    aw, ax, ay, az = a
    bw, bx, by, bz = b
    return np.array(
        [
            aw * bw - ax * bx - ay * by - az * bz,
            aw * bx + ax * bw + ay * bz - az * by,
            aw * by - ax * bz + ay * bw + az * bx,
            aw * bz + ax * by - ay * bx + az * bw,
        ]
    )


# --------------------------------------------------------------------------
# Stage (a): inverse projection (backend.py:78-101)

def inverse_project(depths, confs, frame_ids, pose_q, pose_t, K):
    """One point per positive-depth pixel in the submap (anchor) frame.

    backend.py:85-93: per frame, (vs, us) = nonzero(depth > 0) row-major,
    ray = ((u - cx)/fx*z, (v - cy)/fy*z, z), point = poses[f].apply(ray).
    Returns (points (N,3), conf (N,), frame_ids (N,), pixels (N,2) as (u, v)).
    """
    fx, fy, cx, cy = (float(x) for x in K)
    pts, cs, fids, pix = [], [], [], []
    for f, fid in enumerate(frame_ids):
        depth = np.asarray(depths[f], dtype=float)
        vs, us = np.nonzero(depth > 0)
        z = depth[vs, us]
        rays = np.stack([(us - cx) / fx * z, (vs - cy) / fy * z, z], axis=1)
        pts.append(pose_apply(pose_q[f], pose_t[f], rays))
        cs.append(np.asarray(confs[f], dtype=float)[vs, us])
        fids.append(np.full(len(us), fid, dtype=np.int64))
        pix.append(np.stack([us, vs], axis=1).astype(np.int64))
    if pts:
        return (np.concatenate(pts), np.concatenate(cs), np.concatenate(fids),
                np.concatenate(pix))
    return (np.zeros((0, 3)), np.zeros(0), np.zeros(0, np.int64), np.zeros((0, 2), np.int64))


def frame_points_dense(depth, q, t, K):
    """Dense (H, W, 3) float64 points of one frame; NaN-free, invalid pixels
    carry whatever the formula gives (callers mask with depth > 0).  Same
    arithmetic as inverse_project for the valid pixels."""
    fx, fy, cx, cy = (float(x) for x in K)
    depth = np.asarray(depth, dtype=float)
    h, w = depth.shape
    vs, us = np.meshgrid(np.arange(h), np.arange(w), indexing="ij")
    vs = vs.reshape(-1)
    us = us.reshape(-1)
    z = depth.reshape(-1)
    rays = np.stack([(us - cx) / fx * z, (vs - cy) / fy * z, z], axis=1)
    return pose_apply(q, t, rays).reshape(h, w, 3)


# --------------------------------------------------------------------------
# Stage (b): weighted Umeyama (registration.py)

def normalize_confidences(c):
    """registration.py:28-35 (status instead of exceptions)."""
    c = np.asarray(c, dtype=float)
    if c.size == 0 or not np.any(c > 0):
        return None, STATUS_ALL_ZERO
    if np.any(c < 0):
        return None, STATUS_SHAPE
    return c / c.sum(), STATUS_OK


def align_point_sets(p, q, weights=None, with_scale=True):
    """registration.py:38-102.  Returns (s, quat, t, rms, status)."""
    p = np.asarray(p, dtype=float)
    q = np.asarray(q, dtype=float)
    n = p.shape[0]
    fail = lambda st: (None, None, None, None, st)  # noqa: E731
    if n < 3:
        return fail(STATUS_TOO_FEW)
    if q.shape != p.shape:
        return fail(STATUS_SHAPE)
    if weights is None:
        w = np.full(n, 1.0 / n)
    else:
        w = np.asarray(weights, dtype=float)
        wsum = w.sum()
        if wsum <= 0:
            return fail(STATUS_ALL_ZERO)
        w = w / wsum
    p_bar = w @ p
    q_bar = w @ q
    dp = p - p_bar
    dq = q - q_bar
    cov = (dq * w[:, None]).T @ dp
    u, d, vt = np.linalg.svd(cov)
    src_sv = np.linalg.svd((dp * np.sqrt(w)[:, None]), compute_uv=False)
    if src_sv[1] <= max(1e-12 * src_sv[0], 1e-300):
        return fail(STATUS_DEGENERATE)
    sign = 1.0 if np.linalg.det(u @ vt) >= 0 else -1.0
    flip = np.array([1.0, 1.0, sign])
    r = u @ np.diag(flip) @ vt
    if with_scale:
        var_p = float(w @ np.sum(dp * dp, axis=1))
        s = float((d * flip).sum() / var_p)
        if s <= 0:
            return fail(STATUS_DEGENERATE)
    else:
        s = 1.0
    t = q_bar - s * (r @ p_bar)
    quat = normalize_quat(matrix_to_quat(r))      # Rotation3.from_matrix + __post_init__
    resid = s * (p @ r.T) + t - q
    rms = float(np.sqrt(w @ np.sum(resid * resid, axis=1)))
    return s, quat, t, rms, STATUS_OK


def shared_correspondences(sm, other):
    """mapping.py:138-160 on dense submaps (dicts with depth/conf/frame_ids/
    pose_q/pose_t/K).  Pixel-identity pairs in sm.keyframe order, row-major
    pixel order within a frame (Submap.pixel_rows mapping.py:41-54 inverts the
    np.nonzero compaction of backend.py:87, so rows_a[both] is row-major)."""
    ps, qs, ws = [], [], []
    other_ids = list(other["frame_ids"])
    for fa, kf in enumerate(sm["frame_ids"]):
        if kf not in other_ids:
            continue
        fb = other_ids.index(kf)
        da = np.asarray(sm["depth"][fa], dtype=float)
        db = np.asarray(other["depth"][fb], dtype=float)
        both = (da > 0) & (db > 0)
        pa = frame_points_dense(da, sm["pose_q"][fa], sm["pose_t"][fa], sm["K"])
        pb = frame_points_dense(db, other["pose_q"][fb], other["pose_t"][fb], other["K"])
        ps.append(pa[both])
        qs.append(pb[both])
        ca = np.asarray(sm["conf"][fa], dtype=float)[both]
        cb = np.asarray(other["conf"][fb], dtype=float)[both]
        ws.append(np.minimum(ca, cb))
    if not ps:
        return np.zeros((0, 3)), np.zeros((0, 3)), np.zeros(0)
    return np.concatenate(ps), np.concatenate(qs), np.concatenate(ws)


def registration_edge(sm, other, floor_frac=0.1, min_corr=10):
    """One partner iteration of mapping.py:171-183.

    Returns dict(status, s, q, t, rms, count, keep) where keep is the
    inlier (confidence-floor) mask over the shared correspondences."""
    p, q, w = shared_correspondences(sm, other)
    out = dict(n_pairs=len(p), keep=None, count=0, s=None, q=None, t=None, rms=None)
    if len(p) < min_corr:
        out["status"] = STATUS_SKIP
        return out
    floor = floor_frac * float(w.max())
    keep = w >= floor
    out["keep"] = keep
    if keep.sum() < min_corr:
        out["status"] = STATUS_SKIP
        return out
    s, quat, t, rms, st = align_point_sets(p[keep], q[keep], w[keep])
    out.update(status=st, s=s, q=quat, t=t, rms=rms, count=int(keep.sum()))
    return out


# --------------------------------------------------------------------------
# Stage (c): transform + concatenation (mapping.py:56-57, 332-338) and keys

def world_points(sm, g_s, g_q, g_t):
    """Submap.world_points, mapping.py:56-57: global_pose.apply(cloud.points)."""
    pts, conf, _, _ = inverse_project(sm["depth"], sm["conf"], sm["frame_ids"],
                                      sm["pose_q"], sm["pose_t"], sm["K"])
    return sim3_apply(g_s, g_q, g_t, pts), conf


def fused_cloud(submaps, globals_):
    """Mapping.fused_cloud, mapping.py:332-338 (plain concatenation)."""
    pts, cs = [], []
    for sm, (s, q, t) in zip(submaps, globals_):
        x, c = world_points(sm, s, q, t)
        pts.append(x)
        cs.append(c)
    if not pts:
        return np.zeros((0, 3)), np.zeros(0)
    return np.concatenate(pts), np.concatenate(cs)


def pack(cells):
    """_kernels/_numpy.py:50-55 — three 21-bit fields, offset 2**20."""
    cells = np.asarray(cells, dtype=np.int64)
    return (((cells[..., 0] + PACK_OFFSET) << 42)
            | ((cells[..., 1] + PACK_OFFSET) << 21)
            | (cells[..., 2] + PACK_OFFSET))


def unpack(keys):
    keys = np.asarray(keys, dtype=np.int64)
    m = (1 << 21) - 1
    return np.stack([((keys >> 42) & m) - PACK_OFFSET, ((keys >> 21) & m) - PACK_OFFSET,
                     (keys & m) - PACK_OFFSET], axis=-1)


# --------------------------------------------------------------------------
# Descriptor matching (tracking.py:143-170)

def match_descriptors(desc_a, desc_b, ratio):
    """tracking.py:143-170, verbatim semantics (row-side ratio test only,
    first-index argmin ties, np.partition second value, skipped when M == 1)."""
    desc_a = np.asarray(desc_a, dtype=float)
    desc_b = np.asarray(desc_b, dtype=float)
    if len(desc_a) == 0 or len(desc_b) == 0:
        return []
    sim = desc_a @ desc_b.T
    d2 = np.maximum(2.0 - 2.0 * sim, 0.0)
    best_b = np.argmin(d2, axis=1)
    best_a = np.argmin(d2, axis=0)
    matches = []
    ratio2 = ratio * ratio
    for ia in range(len(desc_a)):
        ib = best_b[ia]
        if best_a[ib] != ia:
            continue
        row = d2[ia]
        d_first = row[ib]
        if len(row) > 1:
            second = np.partition(row, 1)[1]
            if d_first > ratio2 * second:
                continue
        matches.append((ia, int(ib)))
    return matches


def match_descriptors_vec(desc_a, desc_b, ratio):
    """Vectorised form of match_descriptors (same decisions): used by tests
    at sizes where the per-row Python loop is too slow.  Returns an (K, 2)
    int64 array of (ia, ib) ascending in ia."""
    desc_a = np.asarray(desc_a, dtype=float)
    desc_b = np.asarray(desc_b, dtype=float)
    if len(desc_a) == 0 or len(desc_b) == 0:
        return np.zeros((0, 2), np.int64)
    sim = desc_a @ desc_b.T
    d2 = np.maximum(2.0 - 2.0 * sim, 0.0)
    best_b = np.argmin(d2, axis=1)
    best_a = np.argmin(d2, axis=0)
    ia = np.arange(len(desc_a))
    mutual = best_a[best_b] == ia
    if d2.shape[1] > 1:
        second = np.partition(d2, 1, axis=1)[:, 1]
        d_first = d2[ia, best_b]
        ok = ~(d_first > (ratio * ratio) * second)
    else:
        ok = np.ones(len(ia), bool)
    keep = mutual & ok
    return np.stack([ia[keep], best_b[keep]], axis=1).astype(np.int64)


# --------------------------------------------------------------------------
# Global retrieval (loops.py:184-243, database.py:72-80)

def pooled_vector(tokens):
    """KeyframeDatabase.store_embedding pooling, database.py:78-80."""
    pooled = np.asarray(tokens, dtype=float).mean(axis=0)
    n = np.linalg.norm(pooled)
    return pooled / n if n > 0 else pooled


class SimilarityState:
    """SimilarityMatrix (loops.py:156-176) + the ``_admitted`` attribute the
    reference hangs on it (loops.py:212-216)."""

    def __init__(self):
        self.scores = {}
        self.admitted = set()

    @staticmethod
    def key(a, b):
        return (a, b) if a <= b else (b, a)


def update_similarity(state, kf_ids, pooled, stride, exclusion, tau_global, tau_local):
    """loops.py:184-243.  ``kf_ids`` / ``pooled`` are the keyframes that carry
    a pooled vector, in database insertion order (loops.py:197)."""
    order = list(kf_ids)
    index = {kf: i for i, kf in enumerate(order)}
    vec = {kf: np.asarray(pooled[i], dtype=float) for i, kf in enumerate(order)}

    def score(a, b):
        k = SimilarityState.key(a, b)
        cached = state.scores.get(k)
        if cached is not None:
            return cached
        s = float(vec[a] @ vec[b])
        state.scores[k] = s
        return s

    admitted = []
    coarse = [kf for i, kf in enumerate(order) if i % stride == 0]
    for ai in range(len(coarse)):
        for bi in range(ai + 1, len(coarse)):
            a, b = coarse[ai], coarse[bi]
            if abs(index[a] - index[b]) < exclusion:
                continue
            s = score(a, b)
            if s <= tau_global:
                continue
            for da in range(-(stride - 1), stride):
                for db_ in range(-(stride - 1), stride):
                    ia, ib = index[a] + da, index[b] + db_
                    if not (0 <= ia < len(order) and 0 <= ib < len(order)):
                        continue
                    na, nb = order[ia], order[ib]
                    if abs(ia - ib) < exclusion:
                        continue
                    sn = score(na, nb)
                    k = SimilarityState.key(na, nb)
                    if sn > tau_local and k not in state.admitted:
                        state.admitted.add(k)
                        admitted.append((k, sn))
    return admitted
