"""Insert-only timing of the voxel fusion on the bench workload (design
experiments; run on the GPU box, library chosen with EC3R_B200_LIB).

    python tools/fuse_timing.py [--reps 10]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2510_02080_b200 import _lib, mapping  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--keyframes", type=int, default=300)
    args = ap.parse_args()
    dm, sms, desc, _ = bench.build_workload(0, 1, args.keyframes, 1024, "cuda")
    slots = torch.as_tensor(np.concatenate([sm.slots for sm in sms]).astype(np.int32), device="cuda")
    plan = mapping.ChainPlan(sms)
    plan.run(dm.pool)
    vmap = mapping.VoxelMap(0.02, capacity=8 << 20)
    ts = []
    for _ in range(args.reps + 2):
        vmap.clear()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        vmap.insert_frames(dm.pool, slots)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    st = vmap.stats()
    st["voxels"] = vmap.count()
    extra = {}
    # the reduction floor of this insert (ec3r_vhash_diag_log / _replay): its
    # runs logged in issue order, then replayed as pure reductions
    L = _lib.lib()
    cap = int(slots.numel()) * dm.pool.H * dm.pool.W
    runs = torch.empty((cap, 2), dtype=torch.int32, device="cuda")
    n_dev = torch.zeros(1, dtype=torch.int64, device="cuda")
    vmap.clear()
    _lib.check(L.ec3r_vhash_diag_log(vmap._h, _lib.ptr(runs), cap, _lib.ptr(n_dev)), "ec3r_vhash_diag_log")
    vmap.insert_frames(dm.pool, slots)
    extra["runs"] = int(n_dev.item())
    for wc, key in ((1, "replay_ms"), (0, "replay_sums_only_ms")):
        rt = []
        for _ in range(args.reps + 2):
            vmap.clear()
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record()
            _lib.check(L.ec3r_vhash_diag_replay(vmap._h, _lib.ptr(runs), _lib.ptr(n_dev), cap, wc, None), "replay")
            b.record()
            torch.cuda.synchronize()
            rt.append(a.elapsed_time(b))
        extra[key] = float(np.median(rt[2:]))
    print(json.dumps({"lib": os.environ.get("EC3R_B200_LIB", "default"), "insert_ms": float(np.median(ts[2:])),
                      "min_ms": float(np.min(ts[2:])), "stats": {k: int(v) for k, v in st.items()}, **extra}))


if __name__ == "__main__":
    main()
