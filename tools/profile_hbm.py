"""Two C1 builds (1M x 128 SIFT-shaped, 4 shards) through the pipeline, for ncu captures of the
HBM-bound kernels of the second build (prune, reverse, merge fold):
    ncu --set full -k regex:"prune_kernel|indeg_kernel|scatter_kernel|reverse_merge|merge_shard" \\
        --launch-skip 20 --launch-count 5 python tools/profile_hbm.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2605_10135_b200 import api, datagen  # noqa: E402
from paper_2605_10135_b200.pipeline import BuildConfig, build_index  # noqa: E402


def main():
    api.load()
    x = datagen.sift_like(1_000_000, 128, device="cuda")
    cfg = BuildConfig(k=4, L=128, R=64)
    for _ in range(2):
        idx = build_index(x, cfg)
    torch.cuda.synchronize()
    print("sizes", idx.sizes)


if __name__ == "__main__":
    main()
