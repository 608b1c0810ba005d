"""Generate the golden fixtures that pin the oracle to the reference.

Runs the UNMODIFIED reference package (``/root/reference/pkg/src``, imported
read-only) on seeded synthetic inputs and writes its outputs to small .npz
files next to this script.  It only runs in the build container (the GPU box
has no /root/reference); the fixtures are committed so that the oracle tests
(tests/test_oracle_golden.py) and the GPU parity tests can use them anywhere.

Inputs are rounded to float32 (descriptors to bf16-representable values)
before the reference sees their exact float64 upcasts, so the CUDA path —
which stores pointmaps / descriptors in those narrower types — sees
bit-identical inputs.

    python tests/golden/make_golden.py
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF = os.environ.get("EC3R_REFERENCE_SRC", "/root/reference/pkg/src")
sys.path.insert(0, REF)
sys.path.insert(0, os.path.join(os.path.dirname(REF), "tests"))

from submap_slam import backend as rbackend  # noqa: E402
from submap_slam.database import KeyframeDatabase  # noqa: E402
from submap_slam.errors import SubmapSlamError  # noqa: E402
from submap_slam.liegroups import Sim3Transform  # noqa: E402
from submap_slam.loops import FlushBatch, LoopConfig, SimilarityMatrix, update_similarity  # noqa: E402
from submap_slam.mapping import Mapping  # noqa: E402
from submap_slam.registration import align_point_sets  # noqa: E402
from submap_slam.scenesim import TrajectorySpec, WorldConfig, generate_trajectory, generate_world  # noqa: E402
from submap_slam.tracking import match_descriptors  # noqa: E402

from helpers import random_sim3  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def f32(x):
    return np.asarray(x, dtype=np.float32).astype(np.float64)


def bf16(x):
    """Round float64 -> bf16 (nearest-even) -> exact float64 value."""
    a = np.asarray(x, dtype=np.float32)
    u = a.view(np.uint32).astype(np.uint64)
    r = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16
    return r.astype(np.uint32).view(np.float32).astype(np.float64)


# ---------------------------------------------------------------------------
# 1. Umeyama known answers (pkg/tests/test_registration.py:34-154 seeds) plus
#    random problems; outputs of registration.align_point_sets.

def gen_registration():
    cases = []
    rng = np.random.default_rng(20)                      # test_registration.py:35
    gt = Sim3Transform(1.7, random_sim3(rng).rotation, rng.normal(size=3))
    p = rng.normal(size=(10, 3))
    cases.append((p, gt.apply(p), None, True))
    rng = np.random.default_rng(21)                      # :45
    p = rng.normal(size=(8, 3))
    cases.append((p, p.copy(), None, True))
    rng = np.random.default_rng(22)                      # :53
    gt = random_sim3(rng)
    p = rng.normal(size=(50, 3))
    q = gt.apply(p) + rng.normal(size=(50, 3)) * 0.01
    cases.append((p, q, np.ones(50), True))
    cases.append((np.concatenate([p, [[100.0, -100.0, 100.0]]]),
                  np.concatenate([q, [[-100.0, 100.0, -100.0]]]),
                  np.concatenate([np.ones(50), [0.0]]), True))
    p = np.array([[0.0, 0, 0], [1, 0, 0], [2, 0, 0]])    # :75 collinear
    cases.append((p, p + 1.0, None, True))
    d = np.array([0.3, -1.1, 2.7])                        # collinear, general direction
    p = np.outer(np.linspace(-2, 3, 7), d) + np.array([5.0, 1.0, -2.0])
    cases.append((p, p * 1.3 + 0.2, None, True))
    cases.append((np.zeros((2, 3)), np.zeros((2, 3)), None, True))   # :81 too few
    cases.append((np.ones((5, 3)), np.ones((5, 3)), np.zeros(5), True))  # all zero
    rng = np.random.default_rng(23)                      # :89 minimizer problems
    for _ in range(20):
        gt = random_sim3(rng)
        n = int(rng.integers(4, 30))
        p = rng.normal(size=(n, 3))
        w = rng.uniform(0.1, 2.0, size=n)
        q = gt.apply(p) + rng.normal(size=(n, 3)) * 0.05
        cases.append((p, q, w, True))
    rng = np.random.default_rng(26)                      # :134 near planar
    for _ in range(10):
        n = int(rng.integers(4, 20))
        p = rng.normal(size=(n, 3))
        p[:, 2] *= 1e-8
        q = rng.normal(size=(n, 3))
        q[:, 2] *= 1e-8
        cases.append((p, q, None, True))
    rng = np.random.default_rng(1234)                    # large, offset, with_scale False
    for n, off in ((5000, 0.0), (20000, 100.0), (3000, -40.0)):
        gt = random_sim3(rng)
        p = rng.normal(size=(n, 3)) * 2.0 + off
        q = gt.apply(p) + rng.normal(size=(n, 3)) * 0.01
        w = rng.uniform(0.0, 1.0, size=n)
        w[rng.uniform(size=n) < 0.1] = 0.0
        cases.append((p, q, w, True))
    p = rng.normal(size=(40, 3))
    cases.append((p, random_sim3(rng).apply(p), None, False))

    out = {}
    for i, (p, q, w, ws) in enumerate(cases):
        out[f"c{i}_p"] = p
        out[f"c{i}_q"] = q
        out[f"c{i}_w"] = w if w is not None else np.zeros(0)
        out[f"c{i}_hasw"] = np.array(w is not None)
        out[f"c{i}_withscale"] = np.array(ws)
        try:
            tr, rms = align_point_sets(p, q, w, with_scale=ws)
            out[f"c{i}_status"] = np.array("ok")
            out[f"c{i}_s"] = np.array(tr.scale)
            out[f"c{i}_quat"] = np.array(tr.rotation.q)
            out[f"c{i}_t"] = np.array(tr.translation)
            out[f"c{i}_rms"] = np.array(rms)
        except SubmapSlamError as e:
            out[f"c{i}_status"] = np.array(type(e).__name__)
        except ValueError:
            out[f"c{i}_status"] = np.array("ValueError")
    out["n_cases"] = np.array(len(cases))
    np.savez_compressed(os.path.join(OUT, "registration.npz"), **out)
    print("registration:", len(cases), "cases")


# ---------------------------------------------------------------------------
# 2/3. inverse_project, submap registration and fused cloud through the
#      reference Mapping (pkg/tests/test_mapping.py fixture, noisy decode).

class F32Backend(rbackend.SyntheticBackend):
    """Reference SyntheticBackend whose decode output is rounded to float32
    (the storage type of the CUDA path); captures every decode."""

    def __init__(self, *a, **k):
        super().__init__(*a, **k)
        self.captured = []

    def decode(self, embeddings):
        out = super().decode(embeddings)
        out = rbackend.ReconstructionOutput(
            out.frame_ids, f32(out.depths), f32(out.confidences), out.poses,
            out.intrinsics, out.call_index)
        self.captured.append(out)
        return out


def _dense(out):
    return dict(
        depth=out.depths.astype(np.float32),
        conf=out.confidences.astype(np.float32),
        frame_ids=np.array(out.frame_ids, np.int64),
        pose_q=np.array([p.rotation.q for p in out.poses]),
        pose_t=np.array([p.translation for p in out.poses]),
        K=np.array([out.intrinsics.fx, out.intrinsics.fy, out.intrinsics.cx, out.intrinsics.cy]),
    )


def gen_mapping():
    world = generate_world(WorldConfig(room_size=(8.0, 8.0, 4.0), landmark_count=300), 0)
    spec = TrajectorySpec(kind="circle", frame_count=16, radius=2.0, step_bound=1.0)
    traj = generate_trajectory(spec, world)
    cfg = rbackend.SyntheticBackendConfig(depth_resolution=(80, 60), focal=70.0)
    be = F32Backend(world, traj, cfg, seed=100)
    mp = Mapping(be)
    batches = [FlushBatch(new_ids=(0, 1, 2, 3, 4), old_ids=()),
               FlushBatch(new_ids=(5, 6, 7, 8), old_ids=(4,)),
               FlushBatch(new_ids=(9, 10, 11, 12), old_ids=(8,))]
    out = {}
    for j, b in enumerate(batches):
        sm = mp.build_submap(b)
        dec = be.captured[-1]
        d = _dense(dec)
        for k, v in d.items():
            out[f"sm{j}_{k}"] = v
        if j == 0:
            cloud = sm.cloud
            out["ip_points"] = cloud.points
            out["ip_conf"] = cloud.confidences
            out["ip_fids"] = cloud.frame_ids
            out["ip_pixels"] = cloud.pixels
        else:
            other = mp.submaps[j - 1]
            p, q, w = mp._shared_correspondences(sm, other)
            floor = 0.1 * float(w.max())
            out[f"e{j}_p"] = p
            out[f"e{j}_q"] = q
            out[f"e{j}_w"] = w
            out[f"e{j}_keep"] = w >= floor
            edges = mp._registration_edges(sm)
            (sid, tr, info, count, rms), = edges
            out[f"e{j}_partner"] = np.array(sid)
            out[f"e{j}_s"] = np.array(tr.scale)
            out[f"e{j}_quat"] = np.array(tr.rotation.q)
            out[f"e{j}_t"] = np.array(tr.translation)
            out[f"e{j}_rms"] = np.array(rms)
            out[f"e{j}_count"] = np.array(count)
        mp.register_submap(sm)
        g = sm.global_pose
        out[f"sm{j}_gs"] = np.array(g.scale)
        out[f"sm{j}_gq"] = np.array(g.rotation.q)
        out[f"sm{j}_gt"] = np.array(g.translation)
    pts, conf = mp.fused_cloud()
    out["fused_points"] = pts
    out["fused_conf"] = conf
    out["n_submaps"] = np.array(len(batches))
    np.savez_compressed(os.path.join(OUT, "mapping.npz"), **out)
    print("mapping:", len(pts), "fused points")


# ---------------------------------------------------------------------------
# 4. Descriptor matching (tracking.py:143-170) on bf16-representable inputs.

def _desc_pair(rng, n, m, d, sigma, spurious=0.2):
    a = rng.normal(size=(n, d))
    a /= np.linalg.norm(a, axis=1, keepdims=True)
    perm = rng.permutation(n)[:m] if m <= n else rng.integers(0, n, m)
    b = a[perm] + rng.normal(size=(m, d)) * sigma
    b /= np.linalg.norm(b, axis=1, keepdims=True)
    spur = rng.uniform(size=m) < spurious
    fresh = rng.normal(size=(int(spur.sum()), d))
    b[spur] = fresh / np.linalg.norm(fresh, axis=1, keepdims=True)
    return bf16(a), bf16(b)


def gen_match():
    rng = np.random.default_rng(4242)
    cases = []
    cases.append(_desc_pair(rng, 200, 180, 256, 0.10))      # stress noise
    cases.append(_desc_pair(rng, 150, 220, 256, 0.05))      # default noise, N != M
    cases.append(_desc_pair(rng, 97, 61, 64, 0.10))         # synthetic D = 64
    cases.append(_desc_pair(rng, 33, 1, 256, 0.05))         # M == 1: no ratio test
    cases.append((np.eye(60, 80), np.eye(60, 80)))          # test_loops.py:176-177 ties
    cases.append((np.eye(100, 128), np.eye(100, 128)))      # test_loops.py:155
    a, b = _desc_pair(rng, 40, 40, 32, 0.0, spurious=0.0)   # duplicate rows in B
    b[5] = b[7]
    cases.append((a, b))
    cases.append((np.zeros((0, 16)), bf16(rng.normal(size=(5, 16)))))  # empty
    out = {}
    for i, (a, b) in enumerate(cases):
        m = match_descriptors(a, b, 0.8)
        out[f"c{i}_a"] = a.astype(np.float32)
        out[f"c{i}_b"] = b.astype(np.float32)
        out[f"c{i}_matches"] = np.array(m, dtype=np.int64).reshape(-1, 2)
    out["n_cases"] = np.array(len(cases))
    np.savez_compressed(os.path.join(OUT, "match.npz"), **out)
    print("match:", len(cases), "cases")


# ---------------------------------------------------------------------------
# 5. Global retrieval (loops.py:184-243) incl. the admitted-once state.

def _retrieval_case(db, stride, cfg, calls=2):
    matrix = SimilarityMatrix()
    res = [update_similarity(matrix, db, stride, cfg) for _ in range(calls)]
    kf = [k for k in db.ids_in_order() if db.get(k).pooled is not None]
    pooled = np.array([db.get(k).pooled for k in kf])
    items = sorted(matrix.items())
    return kf, pooled, res, items


def gen_retrieval():
    out = {}
    cases = []
    dim = 32                                                 # test_loops.py:218-232
    vecs = [np.eye(dim)[i % dim] for i in range(23)]
    vecs[20] = vecs[0]
    db = KeyframeDatabase()
    for k, v in enumerate(vecs):
        db.store_embedding(k, np.asarray(v, float)[None, :])
    cases.append((db, 5, LoopConfig(buffer_capacity=5)))
    world = generate_world(WorldConfig(room_size=(10.0, 10.0, 4.0), landmark_count=300), 5)
    spec = TrajectorySpec(kind="square-loop", frame_count=41, radius=3.0, step_bound=0.7)
    be = rbackend.SyntheticBackend(world, generate_trajectory(spec, world), seed=6)
    db = KeyframeDatabase()                                  # test_loops.py:247-264
    for fid in range(41):
        db.store_embedding(fid, be.encode(fid).tokens)
    cases.append((db, 5, LoopConfig(buffer_capacity=2)))
    spec = TrajectorySpec(kind="square-loop", frame_count=201, radius=3.0, step_bound=0.7)
    traj = generate_trajectory(spec, world)
    traj = traj + traj[1:100]                                # 1.5 laps: many revisits
    be = rbackend.SyntheticBackend(world, traj, seed=7)
    db = KeyframeDatabase()
    for fid in range(len(traj)):
        if fid % 13 == 5:
            db.ensure(fid)                                   # record without a pooled vector
            continue
        db.store_embedding(fid, be.encode(fid).tokens)
    cases.append((db, 5, LoopConfig(buffer_capacity=5)))
    for i, (db, stride, cfg) in enumerate(cases):
        kf, pooled, res, items = _retrieval_case(db, stride, cfg)
        out[f"c{i}_kf"] = np.array(kf, np.int64)
        out[f"c{i}_pooled"] = pooled
        out[f"c{i}_stride"] = np.array(stride)
        out[f"c{i}_excl"] = np.array(cfg.exclusion_zone())
        out[f"c{i}_tau"] = np.array([cfg.tau_global, cfg.tau_local])
        for c, r in enumerate(res):
            out[f"c{i}_call{c}_pairs"] = np.array([p for p, _ in r], np.int64).reshape(-1, 2)
            out[f"c{i}_call{c}_scores"] = np.array([s for _, s in r], float)
        out[f"c{i}_matrix_keys"] = np.array([k for k, _ in items], np.int64).reshape(-1, 2)
        out[f"c{i}_matrix_vals"] = np.array([v for _, v in items], float)
        print(f"retrieval case {i}: K={len(kf)} admitted={[len(r) for r in res]} matrix={len(items)}")
    out["n_cases"] = np.array(len(cases))
    np.savez_compressed(os.path.join(OUT, "retrieval.npz"), **out)


# ---------------------------------------------------------------------------
# 5. The native-kernel plugin slot (_kernels/_numpy.py): nn_query / raycast
#    on seeded clouds and rays, including exact ties, stray queries past the
#    last ring, empty inputs and axis-parallel rays.

def gen_kernels():
    from submap_slam._kernels import _numpy as rk

    rng = np.random.default_rng(404)
    out = {}
    cases = []
    # uniform cloud, queries inside
    cases.append((rng.uniform(-1, 1, (2000, 3)), rng.uniform(-1, 1, (500, 3)), 0.1))
    # surface-like cloud with exact duplicates; queries on and near it
    u = rng.uniform(0, 2, (1500, 2))
    surf = np.stack([u[:, 0], u[:, 1], 0.3 * np.sin(2 * u[:, 0])], axis=1)
    surf = np.concatenate([surf, surf[:200]])
    q = np.concatenate([surf[:100], surf[100:300] + 0.01 * rng.normal(size=(200, 3))])
    cases.append((surf, q, 0.05))
    # stray queries beyond ring 8 (brute-force path) and far negative coordinates
    cases.append((rng.uniform(-3, -2, (800, 3)), np.concatenate([rng.uniform(-3, -2, (50, 3)),
                                                                 rng.uniform(5, 9, (30, 3))]), 0.02))
    # integer lattice, queries at cell centres / midpoints: many equal distances
    g = np.stack(np.meshgrid(np.arange(6), np.arange(6), np.arange(6), indexing="ij"), -1).reshape(-1, 3) * 0.25
    qq = np.concatenate([g[:40] + 0.125, g[40:80] + np.array([0.125, 0.0, 0.0]), g[80:100]])
    cases.append((g.astype(float), qq, 0.25))
    # float32-representable inputs (the device path's common case)
    cases.append((f32(rng.normal(size=(3000, 3))), f32(rng.normal(size=(700, 3))), 0.15))
    for i, (ref, qry, cell) in enumerate(cases):
        d, ix = rk.nn_query(qry, ref, cell)
        out[f"nn{i}_ref"], out[f"nn{i}_query"], out[f"nn{i}_cell"] = ref, qry, np.float64(cell)
        out[f"nn{i}_dist"], out[f"nn{i}_idx"] = d, ix
    out["n_nn"] = np.int64(len(cases))
    d, ix = rk.nn_query(np.zeros((3, 3)), np.zeros((0, 3)), 0.1)
    out["nn_empty_ref_dist"], out["nn_empty_ref_idx"] = d, ix

    # raycast: room + interior boxes (scenesim.cast_depth call shape)
    room_min, room_max = np.array([0.0, 0.0, 0.0]), np.array([8.0, 8.0, 4.0])
    boxes = [(np.array([2.0, 2.0, 0.0]), np.array([3.0, 3.5, 1.0])),
             (np.array([5.0, 1.0, 0.0]), np.array([6.5, 2.0, 2.0])),
             (np.array([1.0, 6.0, 0.5]), np.array([2.0, 7.0, 1.5]))]
    n = 3000
    org = np.concatenate([rng.uniform([0.5, 0.5, 0.5], [7.5, 7.5, 3.5], (n, 3)),
                          rng.uniform(-2, 10, (500, 3))])
    dirs = rng.normal(size=(len(org), 3))
    dirs[:300, rng.integers(0, 3, 300)] = 0.0          # axis-parallel components
    dirs[300:350] = np.array([1.0, 0.0, 0.0])
    dirs[350:400] = np.array([0.0, -1.0, 0.0])
    dirs[400:420] = 0.0                               # degenerate zero rays
    org[420:440] = np.array([2.0, 2.5, 0.5])           # on a box face
    t = rk.raycast(org, dirs, room_min, room_max, boxes)
    out["rc_origins"], out["rc_dirs"], out["rc_t"] = org, dirs, t
    out["rc_room_min"], out["rc_room_max"] = room_min, room_max
    out["rc_boxes"] = np.stack([np.stack(b) for b in boxes])
    np.savez_compressed(os.path.join(OUT, "kernels.npz"), **out)


# ---------------------------------------------------------------------------
# 6. Local loop candidates (loops.py:114-133 with project_points,
#    geometry.py:87-109): visible counts and decisions on the reference's own
#    test scenes (pkg/tests/test_loops.py:115-157) and a random window.

def gen_local():
    from submap_slam.backend import GroundTruthBackend
    from submap_slam.geometry import project_points
    from submap_slam.loops import LoopConfig, detect_local_candidates
    from submap_slam.tracking import LocalSparseMap, SparseMapPoint

    out = {}
    cases = []
    for seed, frames, stride, extra in ((1, 25, 12, dict(step_bound=0.6)), (2, 60, 3, {})):
        world = generate_world(WorldConfig(room_size=(8.0, 8.0, 4.0), landmark_count=500), seed)
        spec = TrajectorySpec(kind="circle", frame_count=frames, radius=2.0, look_at="forward", **extra)
        traj = generate_trajectory(spec, world)
        be = GroundTruthBackend(world, traj)
        obs0 = be.extract_features(0)
        m = LocalSparseMap()
        lids = obs0.landmark_ids[obs0.landmark_ids >= 0]
        m.insert_batch([SparseMapPoint(i, world.landmarks[l].copy(), world.tags[l].copy(), 1.0, 0)
                        for i, l in enumerate(lids)])
        window = [(i, traj[i]) for i in range(0, frames, stride)]
        cases.append((m.positions(), window, be.intrinsics))
    # random map points, random window poses around the origin
    rng = np.random.default_rng(606)
    pts = rng.uniform([-1.5, -1.5, 1.0], [1.5, 1.5, 5.0], (3000, 3))
    from submap_slam.liegroups import Pose3, Rotation3

    window = []
    for i in range(12):
        q = rng.normal(size=4)
        q[0] = abs(q[0]) + 3.0  # mostly looking down +z, where the points are
        window.append((100 + i, Pose3(Rotation3(q / np.linalg.norm(q)), rng.uniform(-0.5, 0.5, 3))))
    cases.append((pts, window, cases[0][2]))
    cfg = LoopConfig()
    for i, (pos, window, k) in enumerate(cases):
        counts = [int(project_points(p.inverse(), k, pos)[2].sum()) for _, p in window]
        cand = detect_local_candidates(_SM(pos), window, k, cfg)
        out[f"c{i}_pos"] = pos
        out[f"c{i}_kf"] = np.array([kf for kf, _ in window], np.int64)
        out[f"c{i}_poses"] = np.stack([np.concatenate([[1.0], p.rotation.q, p.translation]) for _, p in window])
        out[f"c{i}_intr"] = np.array([k.fx, k.fy, k.cx, k.cy, k.width, k.height], float)
        out[f"c{i}_counts"] = np.array(counts, np.int64)
        out[f"c{i}_cand"] = np.array(cand, np.int64)
    out["n_cases"] = np.int64(len(cases))
    out["tau_p"] = np.float64(cfg.tau_p)
    np.savez_compressed(os.path.join(OUT, "local.npz"), **out)


# --------------------------------------------------------------------------
# §8(f) rank 4: homography RANSAC (geometry.py:594-640) on the reference's own
# test scenes (test_geometry.py:222-280, test_loops.py:144-200) plus random
# mixtures, noisy inliers and degenerate sets

def _homog(h, src):
    sh = np.concatenate([src, np.ones((len(src), 1))], axis=1) @ h.T
    return sh[:, :2] / sh[:, 2:3]


def gen_ransac():
    from submap_slam.geometry import RansacConfig, estimate_homography_ransac

    cases = []  # (src, dst, cfg)
    rng = np.random.default_rng(39)                       # test_homography_exact
    h = np.array([[1.2, 0.1, 5.0], [-0.05, 0.9, -3.0], [1e-4, -2e-4, 1.0]])
    src = rng.uniform(0, 640, size=(60, 2))
    cases.append((src, _homog(h, src), RansacConfig(seed=4)))
    rng = np.random.default_rng(40)                       # test_homography_null_distribution
    for trial in range(20):
        src = rng.uniform(0, 640, size=(100, 2))
        dst = rng.uniform(0, 640, size=(100, 2))
        cases.append((src, dst, RansacConfig(seed=trial)))
    rng = np.random.default_rng(41)                       # test_homography_mixture_ratio
    h = np.array([[1.0, 0.02, 10.0], [0.01, 1.05, -4.0], [0.0, 0.0, 1.0]])
    src = rng.uniform(50, 600, size=(100, 2))
    dst = _homog(h, src)
    bad = rng.choice(100, size=40, replace=False)
    dst[bad] = rng.uniform(0, 640, size=(40, 2))
    cases.append((src, dst, RansacConfig(seed=5)))
    rng = np.random.default_rng(42)                       # test_homography_invariant_to_uniform_rescale
    h = np.array([[0.9, 0.05, 20.0], [-0.02, 1.1, 7.0], [5e-5, 1e-4, 1.0]])
    src = rng.uniform(0, 640, size=(40, 2))
    dst = _homog(h, src)
    cases.append((src, dst, RansacConfig(seed=6)))
    cases.append((src * 3.0, dst * 3.0, RansacConfig(seed=6, pixel_threshold=6.0)))
    for n_in, seed in ((35, 73), (30, 74), (40, 75)):     # test_loops._synthetic_homography_obs
        rng = np.random.default_rng(seed)
        h = np.array([[1.05, 0.02, 4.0], [-0.01, 0.98, -2.0], [1e-5, 0.0, 1.0]])
        src = rng.uniform(20, 600, size=(100, 2))
        dst = _homog(h, src)
        dst[n_in:] = rng.uniform(0, 640, size=(100 - n_in, 2))
        dst[n_in:] += 50.0 * np.sign(dst[n_in:] - 320.0)
        dst[n_in:] = np.clip(dst[n_in:], 0, 640)
        cases.append((src, dst, RansacConfig(seed=3)))
    rng = np.random.default_rng(777)                      # random mixtures with pixel noise
    for n, frac, noise, cfg in ((4, 1.0, 0.0, RansacConfig(seed=1)), (5, 0.8, 0.3, RansacConfig(seed=2)),
                                (8, 0.5, 0.5, RansacConfig(seed=3)), (25, 0.6, 0.8, RansacConfig(seed=4)),
                                (200, 0.3, 0.7, RansacConfig(seed=5)), (200, 0.9, 1.2, RansacConfig(seed=6)),
                                (600, 0.45, 0.6, RansacConfig(seed=7, pixel_threshold=1.5)),
                                (1500, 0.25, 0.5, RansacConfig(seed=8)),
                                (300, 0.15, 0.4, RansacConfig(seed=9, max_iterations=200)),
                                (120, 0.5, 0.5, RansacConfig(seed=10, confidence=0.99, pixel_threshold=3.0))):
        h = np.eye(3) + np.array([[0.1, 0.05, 0], [-0.04, 0.08, 0], [0, 0, 0]]) * rng.normal(size=(3, 3))
        h[:2, 2] = rng.uniform(-30, 30, 2)
        h[2, :2] = rng.uniform(-2e-4, 2e-4, 2)
        src = rng.uniform(0, 640, size=(n, 2))
        dst = _homog(h, src) + noise * rng.normal(size=(n, 2))
        k = int(round(frac * n))
        dst[k:] = rng.uniform(0, 640, size=(n - k, 2))
        cases.append((src, dst, cfg))
    t = np.linspace(0, 600, 30)                           # degenerate: every point on one line
    line = np.stack([t, 0.5 * t + 3.0], axis=1)
    cases.append((line, line + 1.0, RansacConfig(seed=11)))
    dup = np.repeat(rng.uniform(0, 640, size=(3, 2)), 4, axis=0)   # 3 distinct points only
    cases.append((dup, dup * 1.1, RansacConfig(seed=12)))
    out = {}
    for i, (src, dst, cfg) in enumerate(cases):
        res = estimate_homography_ransac(list(zip(src, dst)), cfg)
        out[f"c{i}_src"] = src
        out[f"c{i}_dst"] = dst
        out[f"c{i}_cfg"] = np.array([cfg.pixel_threshold, cfg.confidence, cfg.max_iterations, cfg.seed], float)
        out[f"c{i}_model"] = np.asarray(res.model, float)
        out[f"c{i}_mask"] = np.asarray(res.inlier_mask, bool)
        out[f"c{i}_ratio"] = np.float64(res.inlier_ratio)
    # the reference's hypothesis order: the first draws of rng.choice (geometry.py:612)
    for n, seed in ((4, 0), (60, 4), (100, 7), (1500, 8), (70000, 3)):
        r = np.random.default_rng(seed)
        out[f"draws_{n}_{seed}"] = np.stack([r.choice(n, size=4, replace=False) for _ in range(64)])
    out["n_cases"] = np.int64(len(cases))
    np.savez_compressed(os.path.join(OUT, "ransac.npz"), **out)
    print("ransac:", len(cases), "cases")



def _pnp_scene(rng, n, k, outlier_frac=0.0, noise=0.0, planar=False):
    """test_geometry.py:27-37 (_looking_at_points) + noise / outliers."""
    from helpers import random_pose
    pose = random_pose(rng, max_angle=0.8)
    inv = pose.inverse()
    u = rng.uniform(5, k.width - 6, size=n)
    v = rng.uniform(5, k.height - 6, size=n)
    z = rng.uniform(2.0, 8.0, size=n)
    rays = np.stack([(u - k.cx) / k.fx * z, (v - k.cy) / k.fy * z, z], axis=1)
    pts = rays @ inv.rotation.matrix().T + inv.translation
    if planar:  # points on the world plane z = 0 seen by the camera
        pts[:, 2] = 0.0
        pc = pts @ pose.rotation.matrix().T + pose.translation
        keep = pc[:, 2] > 0.5
        pts, pc = pts[keep], pc[keep]
        u, v = k.fx * pc[:, 0] / pc[:, 2] + k.cx, k.fy * pc[:, 1] / pc[:, 2] + k.cy
    pix = np.stack([u, v], axis=1)
    if noise:
        pix = pix + rng.normal(scale=noise, size=pix.shape)
    if outlier_frac:
        bad = rng.choice(len(pix), size=int(outlier_frac * len(pix)), replace=False)
        pix[bad] = rng.uniform([0, 0], [k.width, k.height], size=(len(bad), 2))
    return pts, pix


def gen_pnp():
    """solve_pnp_ransac (geometry.py:414-474) on the reference's own
    test_geometry.py scenes (:79-133) plus larger noisy / outlier / planar /
    degenerate problems: masks, models and ratios, or the exception."""
    from submap_slam.geometry import CameraIntrinsics, Correspondence2D3D, RansacConfig, solve_pnp_ransac
    K = CameraIntrinsics(fx=100.0, fy=100.0, cx=50.0, cy=50.0, width=100, height=100)
    KV = CameraIntrinsics(fx=500.0, fy=500.0, cx=320.0, cy=240.0, width=640, height=480)
    cases = []
    # the reference's tests, verbatim inputs
    rng = np.random.default_rng(32)
    pts, pix = _pnp_scene(rng, 50, KV)
    cases.append((pts, pix, KV, RansacConfig(seed=1)))
    rng = np.random.default_rng(33)
    pts, pix = _pnp_scene(rng, 50, KV)
    pix = pix + rng.normal(scale=0.5, size=pix.shape)
    for i in rng.choice(50, size=15, replace=False):
        pix[i] = rng.uniform([0, 0], [KV.width, KV.height])
    cases.append((pts, pix, KV, RansacConfig(seed=2)))
    rng = np.random.default_rng(34)
    g_pix, g_pts = [], []
    for i in range(20):
        g_pix.append(rng.uniform(0, 99, size=2))
        g_pts.append(rng.normal(size=3) * 10 + [0, 0, 50])
    cases.append((np.array(g_pts), np.array(g_pix), K, RansacConfig(seed=3, min_inliers=10)))
    rng = np.random.default_rng(35)
    pts, pix = _pnp_scene(rng, 40, KV)
    pix = pix + rng.normal(scale=0.5, size=pix.shape)
    cases.append((pts, pix, KV, RansacConfig(seed=7)))
    cases.append((np.zeros((3, 3)), np.zeros((3, 2)), K, RansacConfig()))  # too few
    # larger problems
    for n, fr, noise, seed in ((200, 0.3, 0.5, 11), (600, 0.5, 0.7, 12), (1500, 0.2, 0.4, 13), (120, 0.6, 1.0, 14)):
        rng = np.random.default_rng(900 + seed)
        pts, pix = _pnp_scene(rng, n, KV, outlier_frac=fr, noise=noise)
        cases.append((pts, pix, KV, RansacConfig(seed=seed)))
    rng = np.random.default_rng(950)
    pts, pix = _pnp_scene(rng, 300, KV, outlier_frac=0.25, noise=0.3, planar=True)
    cases.append((pts, pix, KV, RansacConfig(seed=21)))
    rng = np.random.default_rng(951)
    pts, pix = _pnp_scene(rng, 12, KV)  # exact, few points: many count ties (mean-error tie break)
    cases.append((pts, pix, KV, RansacConfig(seed=22, min_inliers=4)))
    out = {}
    for c, (pts, pix, k, cfg) in enumerate(cases):
        corrs = [Correspondence2D3D(pix[i], pts[i], i) for i in range(len(pts))]
        out[f"c{c}_pts"], out[f"c{c}_pix"] = pts, pix
        out[f"c{c}_K"] = np.array([k.fx, k.fy, k.cx, k.cy, k.width, k.height], np.float64)
        out[f"c{c}_cfg"] = np.array([cfg.seed, cfg.min_inliers, cfg.pixel_threshold, cfg.max_iterations,
                                     cfg.confidence], np.float64)
        try:
            r = solve_pnp_ransac(corrs, k, cfg)
            out[f"c{c}_status"] = np.array("ok")
            out[f"c{c}_mask"] = np.asarray(r.inlier_mask, bool)
            out[f"c{c}_q"] = np.asarray(r.model.rotation.q, np.float64)
            out[f"c{c}_t"] = np.asarray(r.model.translation, np.float64)
            out[f"c{c}_ratio"] = np.float64(r.inlier_ratio)
        except SubmapSlamError as e:
            out[f"c{c}_status"] = np.array(type(e).__name__)
    out["n_cases"] = np.int64(len(cases))
    np.savez_compressed(os.path.join(OUT, "pnp.npz"), **out)
    print("pnp:", len(cases), "cases", [str(out[f"c{c}_status"]) for c in range(len(cases))])


def gen_decode():
    """SyntheticBackend.decode (backend.py:228-281) at 518 x 392 on the
    reference's own world and a circle trajectory (SURVEY §8(d) cfg 1):
    noise-free planes (depth_noise_sigma = 0) for bit-exact checks of the
    device producer, plus the gauge and poses of a noisy backend."""
    from submap_slam.backend import SyntheticBackend, SyntheticBackendConfig
    world = generate_world(WorldConfig(room_size=(8.0, 8.0, 4.0), landmark_count=300), seed=0)
    traj = generate_trajectory(TrajectorySpec(kind="circle", frame_count=16, radius=2.0, step_bound=1.0), world,
                               seed=0)
    out = {}
    for tag, sigma in (("clean", 0.0), ("noisy", 0.01)):
        cfg = SyntheticBackendConfig(depth_resolution=(518, 392), focal=400.0, depth_noise_sigma=sigma)
        be = SyntheticBackend(world, traj, cfg, seed=100)
        for call, ids in enumerate(((0, 1, 2, 3, 4), (4, 5, 6, 7, 8))):
            r = be.decode([rbackend.KeyframeEmbedding(i, np.zeros((1, 1))) for i in ids])
            pfx = f"{tag}{call}_"
            out[pfx + "ids"] = np.array(ids)
            out[pfx + "scale"] = np.float64(be.injected_gauges[-1].scale)
            out[pfx + "pose_q"] = np.stack([p.rotation.q for p in r.poses])
            out[pfx + "pose_t"] = np.stack([p.translation for p in r.poses])
            if sigma == 0.0:
                out[pfx + "depth"] = r.depths.astype(np.float32)
                out[pfx + "conf"] = r.confidences.astype(np.float32)
    out["traj_q"] = np.stack([p.rotation.q for p in traj])
    out["traj_t"] = np.stack([p.translation for p in traj])
    out["room_min"], out["room_max"] = np.asarray(world.room_min, float), np.asarray(world.room_max, float)
    out["boxes"] = np.array([np.concatenate([np.asarray(a, float), np.asarray(b, float)])
                             for a, b in world.config.interior_boxes]).reshape(-1, 6)
    np.savez_compressed(os.path.join(OUT, "decode.npz"), **out)
    print("decode:", {k: v.shape for k, v in out.items() if hasattr(v, "shape")})

class _SM:
    """The sparse map surface detect_local_candidates uses (positions())."""

    def __init__(self, pos):
        self._pos = pos

    def positions(self):
        return self._pos


if __name__ == "__main__":
    gens = [gen_registration, gen_mapping, gen_match, gen_retrieval, gen_kernels, gen_local, gen_ransac, gen_pnp,
            gen_decode]
    want = set(sys.argv[1:])  # e.g. `make_golden.py pnp`: only those fixtures
    for g in gens:
        if not want or g.__name__[4:] in want:
            g()
