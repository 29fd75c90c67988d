"""One shard build (a4-a7) through the C ABI on a synthetic SIFT-shaped shard, for ncu / timing of
the prune and reverse kernels.  python tools/profile_build.py [--m 450000] [--reps 2]"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2605_10135_b200 import api, datagen  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--m", type=int, default=450_000)
    ap.add_argument("--reps", type=int, default=2)
    a = ap.parse_args()
    api.load()
    x = datagen.sift_like(a.m, 128, device="cuda")
    ki, kd = api.scalegann_knn(x, 128)
    torch.cuda.synchronize()
    for _ in range(a.reps):
        t0 = time.perf_counter()
        g, gd = api.scalegann_optimize_from_knn(ki, kd, 64)
        torch.cuda.synchronize()
        print(json.dumps({"m": a.m, "prune+reverse_ms": (time.perf_counter() - t0) * 1e3}))


if __name__ == "__main__":
    main()
