"""a2-a3 partition: the one-CTA reference variant of K2 (SG_PART_SINGLE_CTA=1) and the default
grid-wide variant both bit-exact against the oracle (the variant is read from the environment
once per process, so it runs in a subprocess)."""
import os
import subprocess
import sys

import numpy as np
import pytest

from paper_2605_10135_b200 import datagen

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CODE = r"""
import numpy as np, sys
from paper_2605_10135_b200 import api, datagen
api.load()
x = datagen.sift_like(20000, 32, seed=9)
C = api.scalegann_kmeans(x.cuda(), 5)
home, pd, counts = api.scalegann_partition(x.cuda(), C, omega=3, block_size=1024)
np.savez(sys.argv[1], home=home.cpu().numpy().view(np.uint32), pd=pd.cpu().numpy(), C=C.cpu().numpy())
"""


@pytest.mark.parametrize("single", ["0", "1"])
def test_partition_variants_bit_exact(oracle_mod, tmp_path, single):
    out = tmp_path / "p.npz"
    r = subprocess.run([sys.executable, "-c", CODE, str(out)], cwd=ROOT, capture_output=True, text=True,
                       env=dict(os.environ, SG_PART_SINGLE_CTA=single), timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    g = np.load(out)
    x = datagen.sift_like(20000, 32, seed=9).numpy()
    ref = oracle_mod.partition(x, g["C"], omega=3, block_size=1024)
    assert np.array_equal(g["home"], ref["home"])
    assert np.array_equal(g["pd"], ref["primary_d"])
