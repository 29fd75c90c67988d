"""Helper for tests/test_gpu_knn_large.py: one self-join kNN through the C ABI in a fresh
process (the distance kernel reads its selection switches from the environment once per
process), ids/dists saved to an .npz.
Usage: python -m tests.knn_large_case OUT.npz m L seed kind [precision]"""
import sys

import numpy as np

from paper_2605_10135_b200 import api, datagen


def main():
    out, m, L, seed, kind = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4]), sys.argv[5]
    prec = int(sys.argv[6]) if len(sys.argv) > 6 else api.PREC_AUTO
    api.load()
    x = datagen._make(kind, m, 128 if kind != "deep" else 96, seed, "cpu")
    ids, dd = api.scalegann_knn(x.cuda(), L, precision=prec)
    np.savez(out, ids=ids.cpu().numpy().view(np.uint32), d=dd.cpu().numpy())


if __name__ == "__main__":
    main()
