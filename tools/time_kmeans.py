"""Time a1 (scalegann_kmeans) on SIFT-shaped data for several k (n = 1M x 128)."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2605_10135_b200 import api, datagen  # noqa: E402

api.load()
x = datagen.sift_like(1_000_000, 128, device="cuda")
for k in (4, 16, 32):
    api.scalegann_kmeans(x, k)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    C = api.scalegann_kmeans(x, k)
    torch.cuda.synchronize()
    print(f"k={k} kmeans ms {(time.perf_counter() - t0) * 1e3:.2f}", flush=True)
