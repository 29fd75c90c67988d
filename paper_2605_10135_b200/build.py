"""Build libscalegann.so in-tree with nvcc for sm_100a (no torch JIT cache involved)."""
from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OBJ = os.path.join(HERE, "build", os.environ.get("SG_OBJ_DIR", "obj"))
LIB = os.environ.get("SG_LIB_PATH", os.path.join(HERE, "libscalegann.so"))
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")


def _nccl_dir() -> str:
    """The NCCL that torch loads (the nvidia-nccl wheel), so one NCCL serves the whole process;
    the system NCCL otherwise."""
    try:
        import nvidia.nccl as _n
        d = list(_n.__path__)[0]
        if os.path.exists(os.path.join(d, "include", "nccl.h")):
            return d
    except Exception:
        pass
    return ""


NCCL = _nccl_dir()
NCCL_INC = ["-I", os.path.join(NCCL, "include")] if NCCL else []
NCCL_LINK = (["-Xlinker", os.path.join(NCCL, "lib", "libnccl.so.2"), "-Xlinker", "-rpath=" + os.path.join(NCCL, "lib")]
             if NCCL else ["-lnccl"])
FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17", "--expt-relaxed-constexpr",
    "-Xcompiler", "-fPIC",
    "-I", os.path.join(os.path.dirname(HERE), "include"),
] + NCCL_INC + os.environ.get("SG_NVCC_FLAGS", "").split()


def _deps_mtime() -> float:
    files = glob.glob(os.path.join(CSRC, "*")) + [os.path.join(os.path.dirname(HERE), "include", "scalegann.h"),
                                                  __file__]
    return max(os.path.getmtime(f) for f in files)


def _compile(src: str, verbose: bool) -> str:
    obj = os.path.join(OBJ, os.path.basename(src) + ".o")
    if os.path.exists(obj) and os.path.getmtime(obj) >= _deps_mtime():
        return obj
    cmd = [NVCC, *FLAGS, "-c", src, "-o", obj]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr}")
    if verbose and r.stderr:
        print(r.stderr)
    return obj


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and os.path.exists(LIB) and os.path.getmtime(LIB) >= _deps_mtime():
        return LIB
    os.makedirs(OBJ, exist_ok=True)
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    if force:
        for o in glob.glob(os.path.join(OBJ, "*.o")):
            os.remove(o)
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 4)) as ex:
        objs = list(ex.map(lambda s: _compile(s, verbose), srcs))
    tmp = LIB + ".tmp"
    cmd = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", tmp, *objs, *NCCL_LINK]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stderr}")
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    import sys
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
