"""Parity at the north-star size (C4: BIGANN-shaped 100M x 128 u8, 8 shards), one B200 + the
host's cores, written to gpurun_out/c4_parity.json:
  * the smallest C4 shard's exact kNN (a5) through the same self-join launch the build uses
    (15.8M rows, extrapolated thresholds, 62K row blocks): sampled rows (first, last = ragged
    tail, random) against the oracle's P4 top-128 of the same row over the whole shard;
  * the detour prune (a6) of the sampled rows against the oracle's P5 on the sub-table of the
    sampled rows and their 128 neighbours' rows (all the 2-hop rows P5 reads for them).
    python tools/c4_parity.py [--rows 400]
The oracle runs only here (test tooling), on the data the GPU saw."""
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

SENT = 0xFFFFFFFF


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rows", type=int, default=400)
    ap.add_argument("--n", type=int, default=100_000_000)
    a = ap.parse_args()
    api.load()
    oracle.build()
    t0 = time.perf_counter()
    n, d, k, L, R = a.n, 128, 8, 128, 64
    x = datagen._make("sift_u8", n, d, datagen.DATA_SEED, "cuda")
    C = api.scalegann_kmeans(x, k)
    home, pd, counts = api.scalegann_partition(x, C, omega=2)
    sizes = counts["sizes"]
    s = min(range(k), key=lambda t: (sizes[t], t))
    idmap = api.scalegann_shard_idmap(home, s, m=sizes[s])
    del home, pd
    torch.cuda.empty_cache()
    m = sizes[s]
    t1 = time.perf_counter()
    ki, kd = api.scalegann_knn(x, L, ida=idmap)          # the build's self-join launch
    torch.cuda.synchronize()
    t_knn = time.perf_counter() - t1
    pr, prd = api.scalegann_prune(ki, kd, R)
    torch.cuda.synchronize()
    rng = np.random.default_rng(7)
    rows = sorted(set(range(50)) | set(range(m - 50, m)) | set(rng.choice(m, size=max(0, a.rows - 100),
                                                                           replace=False).tolist()))
    rows = np.array(rows, np.int64)
    rows_t = torch.from_numpy(rows).cuda()
    g_ids = ki[rows_t].cpu().numpy().view(np.uint32)
    g_d = kd[rows_t].cpu().numpy()
    g_pr = pr[rows_t].cpu().numpy().view(np.uint32)
    # sub-table for P5: the sampled rows and every row they list
    need = np.unique(np.concatenate([rows, g_ids[g_ids != SENT].astype(np.int64)]))
    sub_i = ki[torch.from_numpy(need).cuda()].cpu().numpy().view(np.uint32)
    sub_d = kd[torch.from_numpy(need).cuda()].cpu().numpy()
    x_h = x.cpu().numpy()
    im = idmap.cpu().numpy().view(np.uint32)
    del ki, kd, pr, prd, x
    torch.cuda.empty_cache()
    # oracle P4 for the sampled rows: top L+1 with self, minus self
    t2 = time.perf_counter()
    oi, od = oracle.knn(x_h, L + 1, ida=im[rows], xb=x_h, idb=im, self_exclude=False)
    o_ids = np.zeros((len(rows), L), np.uint32)
    o_d = np.zeros((len(rows), L), np.float32)
    for t, r in enumerate(rows):
        keep = oi[t] != r
        if keep.all():
            keep[-1] = False
        o_ids[t], o_d[t] = oi[t][keep], od[t][keep]
    t_oracle = time.perf_counter() - t2
    knn_same = (g_ids == o_ids).all(1) & (g_d == o_d).all(1)
    # oracle P5 on the sub-table (local ids remapped to sub-table rows; rows outside -> SENT)
    v = sub_i.astype(np.int64)
    at = np.minimum(np.searchsorted(need, v), len(need) - 1)
    sub_local = np.where((sub_i != SENT) & (need[at] == v), at, SENT).astype(np.uint32)
    opr, _ = oracle.prune(sub_local, sub_d, R)
    sel = np.searchsorted(need, rows)
    back = need.astype(np.uint32)
    o_pr = np.where(opr[sel] == SENT, SENT, back[np.minimum(opr[sel], len(back) - 1)]).astype(np.uint32)
    prune_same = (g_pr == o_pr).all(1)
    res = {"workload": f"C4 BIGANN-shaped {n}x{d} u8, k={k}: shard {s} ({m} rows, the smallest)",
           "sampled_rows": len(rows), "knn_rows_identical": int(knn_same.sum()),
           "prune_rows_identical": int(prune_same.sum()),
           "sample": "first 50 rows, last 50 rows (ragged tail), random rows",
           "gpu_knn_s": t_knn, "gpu_knn_tflops": 2.0 * m * m * d / t_knn / 1e12, "oracle_s": t_oracle,
           "total_s": time.perf_counter() - t0}
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    json.dump(res, open(os.path.join(ROOT, "gpurun_out", "c4_parity.json"), "w"), indent=1)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
