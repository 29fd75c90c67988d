"""CUDA-event timing of prune (a6) and reverse (a7) alone on a kNN of a SIFT-shaped shard:
python tools/time_prune.py [--m 450000] [--reps 5]"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2605_10135_b200 import api, datagen  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--m", type=int, default=450_000)
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    api.load()
    x = datagen.sift_like(a.m, 128, device="cuda")
    ki, kd = api.scalegann_knn(x, 128)
    out = {}
    for name, fn in (("prune", lambda: api.scalegann_prune(ki, kd, 64)),
                     ("reverse", None)):
        if fn is None:
            pr, prd = api.scalegann_prune(ki, kd, 64)
            fn = lambda: api.scalegann_reverse(pr, prd)  # noqa: E731
        fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        out[name + "_ms"] = e0.elapsed_time(e1) / a.reps
    bytes_prune = a.m * 4 * (128 + 128 * 128 + 64 + 128 + 64)
    out["prune_alg_GBps"] = bytes_prune / (out["prune_ms"] / 1e3) / 1e9
    print(json.dumps({"m": a.m, **out}))


if __name__ == "__main__":
    main()
