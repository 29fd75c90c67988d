"""The beam search (a9, NEXT-1) alone on the C1 graph for ncu: builds the 1M x 128 index, then one
search of 10,000 queries at beam 64 with the ground truth passed in.
    ncu --set full -k regex:beam_kernel -c 1 python tools/profile_search.py"""
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
    idx = build_index(x, BuildConfig(k=4, L=128, R=64))
    q = datagen.sift_like(10_000, 128, seed=datagen.DATA_SEED + datagen.QUERY_SEED_OFFSET, device="cuda")
    gt = torch.zeros(10_000, 10, dtype=torch.int32, device="cuda")
    torch.cuda.synchronize()
    _, _, rec, nd = api.scalegann_search_eval(x, idx.merged, idx.entry, q, topk=10, beam=64, gt=gt, return_ndist=True)
    torch.cuda.synchronize()
    print("distances per query", nd / 10_000)


if __name__ == "__main__":
    main()
