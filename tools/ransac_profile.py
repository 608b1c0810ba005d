"""K9 breakdown: the bench's 64 x 500-match homography batch, timed per phase
(score launches / host walk / refit) with CUDA events and wall clock."""

import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2510_02080_b200 import geometry  # noqa: E402


def problems(n_prob=64, n=500, seed=99):
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(n_prob):
        h = np.eye(3) + 0.05 * rng.normal(size=(3, 3))
        h[2, :2] = rng.uniform(-3e-4, 3e-4, 2)
        h[2, 2] = 1.0
        src = rng.uniform(0, 640, size=(n, 2))
        sh = np.concatenate([src, np.ones((n, 1))], axis=1) @ h.T
        dst = sh[:, :2] / sh[:, 2:3] + 0.5 * rng.normal(size=(n, 2))
        dst[int(0.4 * n):] = rng.uniform(0, 640, size=(n - int(0.4 * n), 2))
        out.append((src, dst))
    return out


if __name__ == "__main__":
    probs = problems()
    seeds = list(range(len(probs)))
    for _ in range(3):
        geometry.estimate_homography_ransac_batch(probs, seeds=seeds)
    torch.cuda.synchronize()
    reps = int(sys.argv[1]) if len(sys.argv) > 1 else 10
    t0 = time.perf_counter()
    for _ in range(reps):
        geometry.estimate_homography_ransac_batch(probs, seeds=seeds)
    torch.cuda.synchronize()
    ms = (time.perf_counter() - t0) * 1e3 / reps
    t0 = time.perf_counter()
    for (s, d), sd in zip(probs, seeds):
        pass
    print({"problems": len(probs), "ms_per_batch": ms, "hypotheses": len(probs) * 1000})
