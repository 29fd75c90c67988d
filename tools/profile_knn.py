"""Run the a5 distance kernel alone on one synthetic shard (for ncu / quick timing).

    python tools/profile_knn.py --m 400000 --L 128 [--reps 3] [--kind sift|gauss]
Prints device time per launch (CUDA events on the launching stream) and achieved TFLOP/s
(algorithmic 2*m^2*d).
"""
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
    ap.add_argument("--m", type=int, default=400_000)
    ap.add_argument("--d", type=int, default=128)
    ap.add_argument("--L", type=int, default=128)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--kind", default="sift")
    ap.add_argument("--precision", type=int, default=0)
    ap.add_argument("--prof", action="store_true")
    a = ap.parse_args()
    api.load()
    x = (datagen.sift_like(a.m, a.d, device="cuda") if a.kind == "sift"
         else datagen.gaussian(a.m, a.d, device="cuda"))
    ws = api.Workspace()
    api.scalegann_knn(x, a.L, precision=a.precision, ws=ws)   # warm-up
    torch.cuda.synchronize()
    api.scalegann_stats_read(reset=True)
    api.scalegann_stats_enable(True)
    for _ in range(a.reps):
        api.scalegann_knn(x, a.L, precision=a.precision, ws=ws)
    torch.cuda.synchronize()
    ms, nl, _ = api.scalegann_stats_read(reset=True)
    if a.prof:
        NW = 18   # warps per CTA of the row-major kernel (producer, MMA, 16 epilogue)
        cnt = torch.zeros(NW * 8, dtype=torch.int64, device="cuda")
        api.scalegann_knn_profile(cnt)
        api.scalegann_knn(x, a.L, precision=a.precision, ws=ws)
        torch.cuda.synchronize()
        api.scalegann_knn_profile(None)
        c = cnt.view(NW, 8).double().cpu()
        names = ["wait", "tmem/full", "compact", "mask", "insert", "final"]
        for w in range(NW):
            print(f"warp {w}: " + " ".join(f"{n}={v / 1e9:.2f}G" for n, v in zip(names, c[w, :6].tolist())))
        # counters are lane-0 sums: lane 0 of each (q, a, stream) warp = one row's insertions per stream
        nrb = a.m / 256.0
        print(f"insertions per row (both streams): {c[2:, 6].sum().item() / (8 * nrb):.1f}"
              f"  insertion-loop iterations per warp-row-block: {c[2:, 7].sum().item() / (16 * nrb):.1f}")
    per = ms / a.reps   # per call (spatial-order pass + main sweep)
    fl = 2.0 * a.m * a.m * a.d
    print(json.dumps({"m": a.m, "d": a.d, "L": a.L, "ms_per_launch": per, "tflops": fl / (per / 1e3) / 1e12}))


if __name__ == "__main__":
    main()
