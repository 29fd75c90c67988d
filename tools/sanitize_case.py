"""A small full pass of the hot path (partition, kNN, prune, reverse, merge, search) for
compute-sanitizer: python tools/sanitize_case.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2605_10135_b200 import api, datagen  # noqa: E402
from paper_2605_10135_b200.pipeline import BuildConfig, build_index  # noqa: E402


def main():
    api.load()
    for kind, d in (("sift", 128), ("deep", 96)):
        x = datagen._make(kind, 3000, d, 9, "cuda")
        idx = build_index(x, BuildConfig(k=2, L=32, R=16, block_size=1024))
        q = datagen._make(kind, 64, d, 10, "cuda")
        api.scalegann_search_eval(x, idx.merged, idx.entry, q, topk=10, beam=32)
    torch.cuda.synchronize()
    print("sanitize case done")


if __name__ == "__main__":
    main()
