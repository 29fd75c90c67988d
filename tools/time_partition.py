"""Time a2-a3 (scalegann_partition): python tools/time_partition.py [n=1M] [k=4] (SIFT-shaped, omega=2)."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2605_10135_b200 import api, datagen  # noqa: E402

api.load()
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
k = int(sys.argv[2]) if len(sys.argv) > 2 else 4
x = datagen.sift_like(n, 128, device="cuda")
C = api.scalegann_kmeans(x, k)
for i in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    home, pd, counts = api.scalegann_partition(x, C, omega=2)
    torch.cuda.synchronize()
    print("partition ms", round((time.perf_counter() - t0) * 1e3, 2), "n", n, "k", k, counts["sizes"][:4], flush=True)
