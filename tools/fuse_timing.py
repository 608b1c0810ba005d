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
    L = _lib.lib()
    if hasattr(L, "ec3r_exp_replay"):
        # EC3R_FI_EXP=6 variant: the insert logged its runs; replay them as
        # pure reductions (the atomic floor of this address stream)
        import ctypes as C
        L.ec3r_exp_log_count.restype = C.c_longlong
        assert L.ec3r_exp_log_alloc(C.c_longlong(80 << 20)) == 0
        vmap.clear()
        vmap.insert_frames(dm.pool, slots)
        torch.cuda.synchronize()
        n_runs = L.ec3r_exp_log_count()
        for wc in (1, 0, 3, 2):
            rt = []
            for _ in range(args.reps + 2):
                vmap.clear()
                a = torch.cuda.Event(enable_timing=True)
                b = torch.cuda.Event(enable_timing=True)
                a.record()
                assert L.ec3r_exp_replay(vmap._h, 148 * 8, wc) == 0
                b.record()
                torch.cuda.synchronize()
                rt.append(a.elapsed_time(b))
            extra[{1: "replay_ms", 0: "replay_sums_only_ms", 3: "replay_addr_only_ms",
                   2: "replay_addr_only_sums_only_ms"}[wc]] = float(np.median(rt[2:]))
        extra["runs"] = int(n_runs)
    print(json.dumps({"lib": os.environ.get("EC3R_B200_LIB", "default"), "insert_ms": float(np.median(ts[2:])),
                      "min_ms": float(np.min(ts[2:])), "stats": {k: int(v) for k, v in st.items()}, **extra}))


if __name__ == "__main__":
    main()
