"""Latency anatomy of small batched matcher calls (design experiment, GPU box):
device time per call (CUDA events, back to back), host time per call (the
Python + ctypes + launch sequence, no sync), and the tensor-core kernel's own
time (library event timers).

    python tools/match_latency.py
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2510_02080_b200 import _lib, synth, tracking  # noqa: E402


def anatomy(name, run, reps=20):
    for _ in range(3):
        run()
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record()
    t0 = time.perf_counter()
    for _ in range(reps):
        run()
    host_ms = (time.perf_counter() - t0) * 1e3 / reps
    b.record()
    torch.cuda.synchronize()
    dev_ms = a.elapsed_time(b) / reps
    _lib.kernel_times()
    _lib.timing_enable(True)
    for _ in range(reps):
        run()
    torch.cuda.synchronize()
    _lib.timing_enable(False)
    kt = {k: v[0] / max(v[1], 1) for k, v in _lib.kernel_times().items()}
    return {"case": name, "call_ms": dev_ms, "host_ms_per_call": host_ms, "kernel_ms": kt}


def main():
    out = []
    A, B, ao, bo = synth.make_descriptor_pairs(7, 4096, 4096, 256, 0.05, seed=7, device="cuda")
    A = A[:4096].repeat(7, 1)
    out.append(anatomy("local_loop_7x4096", lambda: tracking.match_batched_device(A, B, None, None, 0, ao, bo, 0.8)))
    for n in (2048, 8192):
        A, B, ao, bo = synth.make_descriptor_pairs(1, n, n, 256, 0.05, seed=n, device="cuda")
        out.append(anatomy(f"pair_{n}", lambda: tracking.match_batched_device(A, B, None, None, 0, ao, bo, 0.8)))
    for o in out:
        print(json.dumps(o))


if __name__ == "__main__":
    main()
