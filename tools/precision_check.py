"""P4-checker pass rate of the f32 precisions at C2 / C3 density (sampled rows vs the oracle):
python tools/precision_check.py [--m 200000] [--kind deep|text] [--rows 500]"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
from paper_2605_10135_b200 import api, datagen  # noqa: E402
from tests.knn_check import check_knn  # noqa: E402
from tests.test_gpu_knn_large import oracle_rows  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--m", type=int, default=200_000)
    ap.add_argument("--kind", default="deep")
    ap.add_argument("--rows", type=int, default=500)
    a = ap.parse_args()
    api.load()
    oracle.build()
    d = 96 if a.kind == "deep" else 768
    beta = 0.7 if a.kind == "deep" else 1.0
    x = datagen.mixture(a.m, d, beta, seed=35, normalise=True)
    rows = np.array(sorted(np.random.default_rng(1).choice(a.m, size=a.rows, replace=False).tolist()), np.int64)
    oi, od = oracle_rows(oracle, x.numpy(), rows, 128)
    out = {"m": a.m, "kind": a.kind, "rows": a.rows, "median_tau_L": float(np.median(od[:, -1])),
           "median_nn1": float(np.median(od[:, 0]))}
    xc = x.cuda()
    for name, prec in (("tf32", 2), ("tf32x3", 3)):
        ids, dd = api.scalegann_knn(xc, 128, precision=prec)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        ids, dd = api.scalegann_knn(xc, 128, precision=prec)
        torch.cuda.synchronize()
        t = time.perf_counter() - t0
        gi, gd = ids.cpu().numpy().view(np.uint32), dd.cpu().numpy()
        fails, first = check_knn(gi[rows], gd[rows], oi, od, x.numpy()[rows], x.numpy(), self_exclude=False)
        err = np.abs(gd[rows].astype(np.float64) - od.astype(np.float64))
        out[name] = {"rows_failing": fails, "first": first, "max_abs_dist_err": float(err.max()),
                     "seconds": t, "tflops": 2.0 * a.m * a.m * d / t / 1e12}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
