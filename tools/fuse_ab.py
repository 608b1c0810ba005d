"""A/B of the two fusion engines on the bench workload (configs[1] by
default): the binned super-block engine (EC3R_FUSE_ENGINE=binned at map
creation) against the default voxel-block hash.  Checks that keys and counts
are identical and centroids / wsum agree, and times insert + sorted extract of
each with CUDA events.  Run on the GPU box:

    python tools/fuse_ab.py [--keyframes 300] [--reps 10]
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


def run(dm, slots, legacy, reps, U_hint=None):
    if legacy:
        os.environ.pop("EC3R_FUSE_ENGINE", None)
    else:
        os.environ["EC3R_FUSE_ENGINE"] = "binned"
    vmap, out, st = mapping.fuse_slots(dm.pool, slots, 0.02)
    U = int(out[0].numel())
    vmap, out, st = mapping.fuse_slots(dm.pool, slots, 0.02, expected_voxels=U, expected_blocks=st["n_blocks"])
    os.environ.pop("EC3R_FUSE_ENGINE", None)
    bufs = tuple(torch.empty_like(x) for x in out)
    ti, te = [], []
    L = _lib.lib()
    for _ in range(reps + 2):
        vmap.clear()
        a, b, c = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        a.record()
        vmap.insert_frames(dm.pool, slots)
        b.record()
        res = vmap.extract(sort=True, out=bufs)
        c.record()
        torch.cuda.synchronize()
        ti.append(a.elapsed_time(b))
        te.append(b.elapsed_time(c))
    st = vmap.stats()
    return res, {"insert_ms": float(np.median(ti[2:])), "extract_ms": float(np.median(te[2:])),
                 "stats": {k: int(v) for k, v in st.items()}, "voxels": int(res[0].numel())}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--keyframes", type=int, default=300)
    args = ap.parse_args()
    dm, sms, desc, _ = bench.build_workload(0, 1, args.keyframes, 1024, "cuda")
    slots = torch.as_tensor(np.concatenate([sm.slots for sm in sms]).astype(np.int32), device="cuda")
    mapping.ChainPlan(sms).run(dm.pool)
    rb, tb = run(dm, slots, False, args.reps)
    rl, tl = run(dm, slots, True, args.reps)
    kb, kl = rb[0].cpu().numpy(), rl[0].cpu().numpy()
    same_keys = kb.shape == kl.shape and bool(np.array_equal(kb, kl))
    out = {"binned": tb, "legacy": tl, "keys_equal": same_keys}
    if same_keys:
        out["counts_equal"] = bool(torch.equal(rb[3], rl[3]))
        out["max_centroid_diff_m"] = float((rb[1] - rl[1]).abs().max())
        out["max_wsum_rel_diff"] = float(((rb[2] - rl[2]).abs() / rl[2]).max())
    print(json.dumps(out))


if __name__ == "__main__":
    main()
