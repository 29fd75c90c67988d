"""Multi-GPU correctness (needs >= 2 GPUs; skipped otherwise): the pipeline on 2 (and 4) ranks
with the library's NCCL communicator builds owner rows that reassemble to the single-GPU merged
graph byte for byte (P:139, P:242 merge by edge union)."""
import json
import os
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("world", [2, 4])
def test_world_equals_single(tmp_path, world):
    if torch.cuda.device_count() < world:
        pytest.skip(f"needs {world} GPUs")
    out = tmp_path / "r.json"
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(29500 + world), "tests/dist_world_case.py", str(out),
           "40000", str(2 * world)]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    res = json.load(open(out))
    assert res["home_equal"] and res["entry_equal"], res
    assert res["ids_equal"] and res["dists_equal"], res
