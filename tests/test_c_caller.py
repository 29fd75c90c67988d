"""The C ABI alone builds an index ("a C-only caller can build a multi-GPU
index"): examples/c_build.c drives a1-a8 through include/scalegann.h, with a file carrying the
communicator's unique id.  CPU: it compiles and links against the library.  GPU: its merged rows
equal the Python pipeline's on the same data (world 1), and on 2 GPUs the two ranks' owner rows
reassemble to the same graph."""
import os
import subprocess

import numpy as np
import pytest
import torch

from paper_2605_10135_b200 import datagen

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _build():
    r = subprocess.run(["bash", "examples/build.sh"], cwd=ROOT, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    return os.path.join(ROOT, "examples", "c_build")


def test_c_caller_compiles():
    from paper_2605_10135_b200 import build
    build.build()
    assert os.path.exists(_build())


@pytest.mark.gpu
@pytest.mark.parametrize("world", [1, 2])
def test_c_caller_equals_python(tmp_path, world):
    if torch.cuda.device_count() < world:
        pytest.skip(f"needs {world} GPUs")
    from paper_2605_10135_b200 import api
    from paper_2605_10135_b200.pipeline import BuildConfig, build_index
    exe = _build()
    n, d, k = 20_000, 64, 3
    x = datagen.sift_like(n, d, seed=91)
    data = tmp_path / "x.bin"
    x.numpy().astype(np.float32).tofile(data)
    uid, out = tmp_path / "uid", tmp_path / "out.bin"
    procs = [subprocess.Popen([exe, str(data), str(n), str(d), str(k), str(r), str(world), str(uid), str(out)],
                              stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True) for r in range(world)]
    for p in procs:
        o, e = p.communicate(timeout=600)
        assert p.returncode == 0, e[-2000:]
    api.load()
    idx = build_index(x.cuda(), BuildConfig(k=k, L=64, R=32))
    ref = idx.merged.cpu().numpy().view(np.uint32)
    if world == 1:
        got = np.fromfile(f"{out}.0", np.uint32).reshape(n, 32)
        assert np.array_equal(got, ref)
    else:
        from paper_2605_10135_b200.pipeline import lpt_owner
        owner = np.array(lpt_owner(idx.sizes, world))
        prim_owner = owner[idx.home[:, 0].long().cpu().numpy()]
        full = np.zeros((n, 32), np.uint32)
        for r in range(world):
            full[prim_owner == r] = np.fromfile(f"{out}.{r}", np.uint32).reshape(-1, 32)
        assert np.array_equal(full, ref)
