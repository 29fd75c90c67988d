"""Helper for tests/test_gpu_knn_modes.py: run one kNN through the C ABI in a fresh process
(the distance kernel reads its tuning switches from the environment once per process) and
save ids/dists to an .npz.  Usage: python -m tests.knn_env_case OUT.npz m L seed [u8]"""
import sys

import numpy as np

from paper_2605_10135_b200 import api, datagen


def main():
    out, m, L, seed = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
    as_u8 = len(sys.argv) > 5 and sys.argv[5] == "u8"
    api.load()
    x = datagen.sift_like(m, 128, seed=seed, as_u8=as_u8)
    ids, dd = api.scalegann_knn(x.cuda(), L)
    np.savez(out, ids=ids.cpu().numpy().view(np.uint32), d=dd.cpu().numpy())


if __name__ == "__main__":
    main()
