"""Per-shard timing of the build on the bench workload (C1): partition, then each shard's
distance kernel timed alone with the diagnostics counters."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2605_10135_b200 import api, datagen  # noqa: E402


def main():
    api.load()
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
    k = 4
    x = datagen.sift_like(n, 128, device="cuda")
    C = api.scalegann_kmeans(x, k)
    home, pd, counts = api.scalegann_partition(x, C, omega=2)
    ws = api.Workspace()
    for s in range(k):
        idm = api.scalegann_shard_idmap(home, s, m=counts["sizes"][s])
        api.scalegann_knn(x, 128, ida=idm, ws=ws)   # warm-up
        torch.cuda.synchronize()
        cnt = torch.zeros(80, dtype=torch.int64, device="cuda")
        api.scalegann_stats_read(reset=True)
        api.scalegann_stats_enable(True)
        api.scalegann_knn(x, 128, ida=idm, ws=ws)
        torch.cuda.synchronize()
        ms, nl, _ = api.scalegann_stats_read(reset=True)
        api.scalegann_knn_profile(cnt)
        api.scalegann_knn(x, 128, ida=idm, ws=ws)
        torch.cuda.synchronize()
        api.scalegann_knn_profile(None)
        c = cnt.view(10, 8).double().cpu()
        m = counts["sizes"][s]
        ins = c[2:, 6].sum().item() / (8 * 148 * max(1, (m // 256) // 148))
        names = ["wait", "tmem", "compact", "mask", "insert", "final"]
        e = c[2:, :6].mean(0)
        print(json.dumps({"shard": s, "m": m, "ms_total(order+main)": ms, "launches": nl,
                          "tflops_main_est": 2.0 * m * m * 128 / (ms / 1e3) / 1e12,
                          "insertions_per_row": ins,
                          "epi_G": {nm: round(v / 1e9, 2) for nm, v in zip(names, e.tolist())}}))


if __name__ == "__main__":
    main()
