"""a5 kNN under every selection mode of the distance kernel, bit-exact against the oracle on
integer (F16_EXACT) data.  Each case runs in its own process because the kernel reads its
switches from the environment once:
  * default: extrapolated thresholds (columns in id order) + device-side fallback;
  * SG_KNN_ALPHA=5 / BETA=1: thresholds far too tight, so most rows take the fallback launch;
  * SG_KNN_ALPHA=0: plain rank-L thresholds;
  * SG_KNN_C=256 / 1024 and SG_KNN_KEEP=1: candidate-buffer sizes and exact compaction;
  * SG_KNN_ORDER=1: spatially ordered shard + rotated column sweep;
  * SG_KNN_T=1: the transposed (column-per-lane, ballot) kernel instead of the row-per-lane one.
"""
import os
import subprocess
import sys

import numpy as np
import pytest

from paper_2605_10135_b200 import datagen

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

MODES = {
    "default": {},
    "fallback_most_rows": {"SG_KNN_ALPHA": "5", "SG_KNN_BETA": "1"},
    "plain_rank_L": {"SG_KNN_ALPHA": "0"},
    "C256_exact": {"SG_KNN_C": "256", "SG_KNN_KEEP": "1"},
    "C1024": {"SG_KNN_C": "1024"},
    "spatial_order": {"SG_KNN_ORDER": "1", "SG_ORDER_GROUP_ROWS": "128"},
    "transposed": {"SG_KNN_T": "1"},
    "transposed_fallback": {"SG_KNN_T": "1", "SG_KNN_ALPHA": "5", "SG_KNN_BETA": "1"},
    "transposed_exact": {"SG_KNN_T": "1", "SG_KNN_ALPHA": "0"},
    "transposed_spatial": {"SG_KNN_T": "1", "SG_KNN_ORDER": "1", "SG_ORDER_GROUP_ROWS": "128"},
}


@pytest.mark.parametrize("mode", list(MODES))
@pytest.mark.parametrize("m,L,seed", [(5000, 128, 3), (2100, 64, 4), (3000, 256, 5)])
def test_knn_modes_bit_exact(oracle_mod, tmp_path, mode, m, L, seed):
    out = tmp_path / "r.npz"
    env = dict(os.environ, **MODES[mode], SG_KNN_REPORT="1")
    r = subprocess.run([sys.executable, "-m", "tests.knn_env_case", str(out), str(m), str(L), str(seed)],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    g = np.load(out)
    x = datagen.sift_like(m, 128, seed=seed)
    oi, od = oracle_mod.knn(x.numpy(), L)
    assert np.array_equal(g["ids"], oi), f"{mode}: ids differ in {(g['ids'] != oi).any(1).sum()} rows"
    assert np.array_equal(g["d"], od)


def test_knn_duplicates_fallback(oracle_mod, tmp_path):
    """Many exact duplicates (ties at the threshold) with thresholds forced too tight."""
    out = tmp_path / "r.npz"
    env = dict(os.environ, SG_KNN_ALPHA="20", SG_KNN_BETA="1", SG_KNN_C="256")
    code = ("import numpy as np, sys; from paper_2605_10135_b200 import api, datagen; api.load();"
            "x = datagen.sift_like(3000, 128, seed=21); x[1000:2000] = x[0:1000];"
            "i, d = api.scalegann_knn(x.cuda(), 128);"
            f"np.savez(r'{out}', ids=i.cpu().numpy().view(np.uint32), d=d.cpu().numpy())")
    r = subprocess.run([sys.executable, "-c", code], cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    g = np.load(out)
    x = datagen.sift_like(3000, 128, seed=21)
    x[1000:2000] = x[0:1000]
    oi, od = oracle_mod.knn(x.numpy(), 128)
    assert np.array_equal(g["ids"], oi) and np.array_equal(g["d"], od)
