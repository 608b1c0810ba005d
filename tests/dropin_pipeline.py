"""End-to-end drop-in check (run by tests/test_gpu_reference_suite.py in a
subprocess, with the reference importable from baseline/_ref): the
reference's own Pipeline (pipeline.py:94-553, unmodified) runs one synthetic
sequence twice -- first on its numpy path, then with the hot-path names
rebound to the B200 package (binding.install(): Mapping, align_point_sets,
match_descriptors, update_similarity, detect_local_candidates,
verify_candidate, inverse_project, ...).  Decisions (keyframes, submaps,
every pipeline event) must be identical (float fields of event records
within 1e-5), poses within 1e-5 and the fused cloud (mapping.py:332-338
concatenation) within 1e-6 m / confidences within float32 rounding; the B200 map's
fused_cloud(voxel=0.02) is checked against the declared voxel rule.
Prints one JSON line; exit 0 = pass."""

import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def run(frames: int):
    from submap_slam.backend import make_backend
    from submap_slam.config import PipelineConfig
    from submap_slam.pipeline import run_pipeline
    from submap_slam.scenesim import TrajectorySpec, generate_trajectory, generate_world

    cfg = PipelineConfig(trajectory=TrajectorySpec(kind="circle", frame_count=frames, radius=2.0))
    world = generate_world(cfg.world, cfg.world_seed)
    traj = generate_trajectory(cfg.trajectory, world, seed=cfg.world_seed)
    t0 = time.perf_counter()
    art = run_pipeline(cfg, make_backend(cfg.backend_name, world, traj, cfg.backend, seed=cfg.seed))
    return art, time.perf_counter() - t0


def events_of(art):
    return [repr(e) for e in art.events]


def event_equal(a: str, b: str) -> bool:
    """Same event kind, frame, decision and integer fields; float fields
    (residuals, ratios, scores) within 1e-5 relative or 1e-12 absolute."""
    import re

    num = re.compile(r"[-+]?(?:\d+\.\d*|\.\d+|\d+)(?:[eE][-+]?\d+)?")
    if num.sub("#", a) != num.sub("#", b):
        return False
    for x, y in zip(num.findall(a), num.findall(b)):
        if x == y:
            continue
        fx, fy = float(x), float(y)
        if not abs(fx - fy) <= max(1e-12, 1e-5 * max(abs(fx), abs(fy))):
            return False
    return True


def main():
    frames = int(sys.argv[1]) if len(sys.argv) > 1 else 60
    ref_art, t_ref = run(frames)
    from paper_2510_02080_b200 import binding

    bound = binding.install()
    b2_art, t_b2 = run(frames)
    out = {"frames": frames, "rebound": len(bound), "t_reference_s": t_ref, "t_b200_s": t_b2,
           "keyframes": [ref_art.keyframe_count, b2_art.keyframe_count],
           "submaps": [ref_art.submap_count, b2_art.submap_count],
           "aborted": [ref_art.aborted, b2_art.aborted]}
    ok = (ref_art.keyframe_count == b2_art.keyframe_count and ref_art.submap_count == b2_art.submap_count
          and ref_art.aborted == b2_art.aborted)
    ev_r, ev_b = events_of(ref_art), events_of(b2_art)
    out["events"] = len(ev_r)
    out["events_equal"] = len(ev_r) == len(ev_b) and all(event_equal(a, b) for a, b in zip(ev_r, ev_b))
    out["events_identical_text"] = ev_r == ev_b
    if not out["events_equal"]:
        diff = [i for i, (a, b) in enumerate(zip(ev_r, ev_b)) if not event_equal(a, b)]
        out["first_event_diff"] = [ev_r[diff[0]], ev_b[diff[0]]] if diff else [len(ev_r), len(ev_b)]
    ok &= out["events_equal"]
    pr = np.stack([np.concatenate([p.rotation.q, p.translation]) for p in ref_art.trajectory.poses])
    pb = np.stack([np.concatenate([p.rotation.q, p.translation]) for p in b2_art.trajectory.poses])
    qsign = np.sign(np.sum(pr[:, :4] * pb[:, :4], axis=1, keepdims=True))
    out["max_pose_diff"] = float(np.max(np.abs(np.concatenate([pr[:, :4] - qsign * pb[:, :4], pr[:, 4:] - pb[:, 4:]],
                                                                 axis=1))))
    ok &= out["max_pose_diff"] < 1e-5
    cr, cb = ref_art.cloud_points, b2_art.cloud_points
    out["cloud_points"] = [len(cr), len(cb)]
    ok &= len(cr) == len(cb)
    if len(cr) == len(cb):
        out["max_cloud_diff_m"] = float(np.max(np.abs(cr - cb))) if len(cr) else 0.0
        ok &= out["max_cloud_diff_m"] < 1e-6
        # the B200 pool keeps planes as float32 (8 B/px): confidences round-trip
        # through float32, points come from float32 depths
        dc = np.abs(ref_art.cloud_confidences - b2_art.cloud_confidences)
        out["max_conf_rel_diff"] = float(np.max(dc / np.maximum(np.abs(ref_art.cloud_confidences), 1e-30)))
        ok &= out["max_conf_rel_diff"] < 1e-7
    # the B200 map's voxel fusion against the declared rule on the same cloud
    from oracle import fuse as ofuse

    vox = b2_art.mapping.fused_cloud(voxel=0.02)
    o = ofuse.fuse_points(cb, b2_art.cloud_confidences, 0.02)
    out["voxels"] = int(len(vox["keys"]))
    vok = (np.array_equal(vox["keys"], o["keys"]) and np.array_equal(vox["count"], o["count"])
           and float(np.max(np.abs(vox["centroid"] - o["centroid"]))) < 1e-4)
    out["voxels_ok"] = bool(vok)
    ok &= vok
    out["ok"] = bool(ok)
    print(json.dumps(out))
    return 0 if ok else 1


if __name__ == "__main__":
    sys.exit(main())
