"""a5 kNN parity where the persistent distance kernel runs MORE row blocks than it has CTAs
(148 CTAs x 256 rows = 37,888 rows for f16, 148 x 128 = 18,944 for TF32): the A-block reload,
the TMEM-buffer phase carried across row blocks and the reuse of the candidate buffers are only
exercised there (VERDICT r1 "what's weak" #2).  Sampled rows (first and last row blocks, the
ragged tail, and random rows) are compared with the oracle's exact P4 top-L of the same row
against the whole set:
  * integer data (F16_EXACT): ids and dists identical, in the default (extrapolated), fallback
    (thresholds far too tight) and plain rank-L modes, and for u8 input;
  * f32 data (TF32 / TF32X3): the P4 tolerance checker (tests/knn_check.py).
"""
import os
import subprocess
import sys

import numpy as np
import pytest

from paper_2605_10135_b200 import datagen
from tests.knn_check import check_knn

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SENT = 0xFFFFFFFF

MODES = {
    "default": {},
    "fallback_most_rows": {"SG_KNN_ALPHA": "5", "SG_KNN_BETA": "1"},
    "plain_rank_L": {"SG_KNN_ALPHA": "0"},
    "cta_pair": {"SG_KNN_2CTA": "1"},                       # opt-in cta_group::2 kernel (knn_tc2.cu)
    "cta_pair_fallback": {"SG_KNN_2CTA": "1", "SG_KNN_ALPHA": "5", "SG_KNN_BETA": "1"},
}


def _run(tmp_path, env_extra, m, L, seed, kind, prec=0):
    out = tmp_path / "r.npz"
    env = dict(os.environ, **env_extra, SG_KNN_REPORT="1")
    r = subprocess.run([sys.executable, "-m", "tests.knn_large_case", str(out), str(m), str(L), str(seed), kind,
                        str(prec)], cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    g = np.load(out)
    return g["ids"], g["d"], r.stderr


def sample_rows(m, n_random, seed, block=256):
    rng = np.random.default_rng(seed)
    fixed = list(range(0, min(m, 300))) + list(range(max(0, m - 700), m))   # first blocks + ragged tail
    fixed += list(range(148 * block - 64, min(m, 148 * block + 64)))          # the second row block of CTA 0
    rnd = rng.choice(m, size=min(m, n_random), replace=False).tolist()
    return np.array(sorted(set(fixed + rnd)), np.int64)


def oracle_rows(oracle_mod, x, rows, L):
    """Exact top-L of each sampled row against the whole set, self excluded: the top L+1 with the
    self column included, minus self (if self is not among them, >= L+1 exact duplicates with
    lower ids precede it and the first L are the answer)."""
    ids, dd = oracle_mod.knn(x, L + 1, ida=rows.astype(np.uint32), xb=x, self_exclude=False)
    out_i = np.zeros((len(rows), L), np.uint32)
    out_d = np.zeros((len(rows), L), np.float32)
    for t, r in enumerate(rows):
        keep = ids[t] != r
        if keep.all():
            keep[-1] = False
        out_i[t] = ids[t][keep]
        out_d[t] = dd[t][keep]
    return out_i, out_d


@pytest.mark.parametrize("mode", list(MODES))
def test_knn_40k_rows_bit_exact(oracle_mod, tmp_path, mode):
    m, L, seed = 40_000, 128, 31
    gi, gd, log = _run(tmp_path, MODES[mode], m, L, seed, "sift")
    x = datagen.sift_like(m, 128, seed=seed).numpy()
    rows = sample_rows(m, 1500, seed)
    oi, od = oracle_rows(oracle_mod, x, rows, L)
    bad = np.nonzero((gi[rows] != oi).any(1) | (gd[rows] != od).any(1))[0]
    assert len(bad) == 0, f"{mode}: {len(bad)} of {len(rows)} sampled rows differ, first row {rows[bad[0]]}; {log[-500:]}"


def test_knn_80k_rows_u8_bit_exact(oracle_mod, tmp_path):
    """u8 input, ~2.1 row blocks per CTA (3 on some CTAs)."""
    m, L, seed = 80_000, 128, 32
    gi, gd, log = _run(tmp_path, {}, m, L, seed, "sift_u8")
    x = datagen.sift_like(m, 128, seed=seed, as_u8=True).numpy()
    rows = sample_rows(m, 1500, seed)
    oi, od = oracle_rows(oracle_mod, x, rows, L)
    bad = np.nonzero((gi[rows] != oi).any(1) | (gd[rows] != od).any(1))[0]
    assert len(bad) == 0, f"{len(bad)} of {len(rows)} sampled rows differ, first row {rows[bad[0]]}; {log[-500:]}"


@pytest.mark.parametrize("prec,mode", [(2, "default"), (2, "fallback_most_rows"), (3, "default")])
def test_knn_40k_rows_f32_tolerance(oracle_mod, tmp_path, prec, mode):
    """DEEP-shaped L2-normalised 96-d f32 (C2's shape), TF32 (RB = 128: 313 row blocks) and
    TF32X3, against the P4 checker on sampled rows."""
    m, L, seed = 40_000, 128, 33
    gi, gd, log = _run(tmp_path, MODES[mode], m, L, seed, "deep", prec)
    x = datagen.mixture(m, 96, 0.7, seed=seed, normalise=True).numpy()
    rows = sample_rows(m, 600, seed, block=128)
    oi, od = oracle_rows(oracle_mod, x, rows, L)
    assert all(r not in gi[r] for r in rows)    # no self loops
    fails, first = check_knn(gi[rows], gd[rows], oi, od, x[rows], x, self_exclude=False)
    assert fails == 0, f"{fails} of {len(rows)} rows fail the P4 checker: {first}"


@pytest.mark.parametrize("prec", [0, 3])
def test_knn_c2_density_f32_p4_checker(oracle_mod, tmp_path, prec):
    """C2-shaped density (DEEP-like 96-d L2-normalised, 200,000 rows): 2,000
    sampled rows pass the P4 checker with AUTO (which must pick an accurate enough precision for
    non-integer data) and with TF32X3."""
    m, L, seed = 200_000, 128, 35
    gi, gd, log = _run(tmp_path, {}, m, L, seed, "deep", prec)
    x = datagen.mixture(m, 96, 0.7, seed=seed, normalise=True).numpy()
    rng = np.random.default_rng(seed)
    rows = np.array(sorted(rng.choice(m, size=2000, replace=False).tolist()), np.int64)
    oi, od = oracle_rows(oracle_mod, x, rows, L)
    fails, first = check_knn(gi[rows], gd[rows], oi, od, x[rows], x, self_exclude=False)
    assert fails == 0, f"precision {prec}: {fails} of {len(rows)} rows fail the P4 checker: {first}"
