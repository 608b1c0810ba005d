"""Reduction-order probe for the fusion insert (design experiment, GPU box).

The insert's runs are logged in issue order (ec3r_vhash_diag_log) and then
replayed as pure reductions (ec3r_vhash_diag_replay) in several orders, to
bound what reordering / deduplicating a warp's or a CTA's runs before their
global reductions could buy:

  logged        the kernel's own issue order (the live reduction floor)
  sort<G>       runs sorted by voxel inside consecutive groups of G
  dedup<G>      ... and equal voxels of a group merged into one reduction
  dedup_all     one reduction per voxel (lower bound)

    python tools/fuse_order_probe.py [--keyframes 300] [--reps 10]
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


def grouped(runs, n, g, dedup):
    r = runs[:n].long()
    vid, cnt = r[:, 0] & 0xFFFFFFFF, r[:, 1]
    grp = torch.arange(n, device=r.device) // g if g else torch.zeros(n, dtype=torch.long, device=r.device)
    key = (grp << 32) | vid
    key, order = torch.sort(key)
    cnt = cnt[order]
    if dedup:
        key, inv = torch.unique_consecutive(key, return_inverse=True)
        c2 = torch.zeros(key.numel(), dtype=torch.long, device=r.device)
        c2.index_add_(0, inv, cnt)
        cnt = c2
    out = torch.stack([(key & 0xFFFFFFFF), cnt], 1).to(torch.int64)
    out = torch.where(out >= 2**31, out - 2**32, out).to(torch.int32).contiguous()
    return out, out.shape[0]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--keyframes", type=int, default=300)
    args = ap.parse_args()
    dm, sms, desc, _ = bench.build_workload(0, 1, args.keyframes, 1024, "cuda")
    del desc
    slots = torch.as_tensor(np.concatenate([sm.slots for sm in sms]).astype(np.int32), device="cuda")
    plan = mapping.ChainPlan(sms)
    plan.run(dm.pool)
    vmap = mapping.VoxelMap(0.02, capacity=8 << 20)
    L = _lib.lib()
    cap = int(slots.numel()) * dm.pool.H * dm.pool.W
    runs = torch.empty((cap, 2), dtype=torch.int32, device="cuda")
    n_dev = torch.zeros(1, dtype=torch.int64, device="cuda")
    vmap.clear()
    _lib.check(L.ec3r_vhash_diag_log(vmap._h, _lib.ptr(runs), cap, _lib.ptr(n_dev)), "ec3r_vhash_diag_log")
    vmap.insert_frames(dm.pool, slots)
    torch.cuda.synchronize()
    n = int(n_dev.item())

    def replay(rr, nn, with_count):
        nd = torch.tensor([nn], dtype=torch.int64, device="cuda")
        ts = []
        for _ in range(args.reps + 2):
            vmap.clear()
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record()
            _lib.check(L.ec3r_vhash_diag_replay(vmap._h, _lib.ptr(rr), _lib.ptr(nd), nn, with_count, None), "replay")
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        return float(np.median(ts[2:]))

    out = {"keyframes": args.keyframes, "points": int(vmap.stats().get("points", 0)) if hasattr(vmap, "stats") else None,
           "runs": n}
    rows = [("logged", runs, n)]
    for g in (32, 128, 1024, 8192):
        rows.append((f"sort{g}",) + grouped(runs, n, g, False))
        rows.append((f"dedup{g}",) + grouped(runs, n, g, True))
    rows.append(("dedup_all",) + grouped(runs, n, 0, True))
    for name, rr, nn in rows:
        out[name] = {"n": int(nn), "ms": replay(rr, nn, 1), "sums_only_ms": replay(rr, nn, 0)}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
