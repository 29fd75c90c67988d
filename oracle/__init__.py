"""CPU oracle for the ScaleGANN hot path — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` leg and ``--impl reference``) may import this package.  It
wraps ``oracle/oracle.c`` (plain C, see its header for the paper passage each
function follows and what pins it) through ctypes with numpy arrays.  It shares
no code with ``paper_2605_10135_b200`` and never imports it.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
SENT = 0xFFFFFFFF
_lib = None


def build(force: bool = False) -> str:
    """Compile oracle.c with gcc (building the checker is not using it)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-std=gnu11", "-fPIC", "-shared", "-ffp-contract=off", "-fopenmp",
               "-o", _LIB, _SRC, "-lm"]
        subprocess.run(cmd, check=True)
    return _LIB


def _load():
    global _lib
    if _lib is None:
        build()
        _lib = ctypes.CDLL(_LIB)
        u64, u32, i32, f32, vp = (ctypes.c_uint64, ctypes.c_uint32, ctypes.c_int, ctypes.c_float,
                                  ctypes.c_void_p)
        _lib.oracle_kmeans.argtypes = [vp, i32, u64, u32, u32, u64, u32, u32, vp, vp]
        _lib.oracle_kmeans.restype = i32
        _lib.oracle_kmeans_distortion.argtypes = [vp, i32, u64, u32, u32, u32, vp]
        _lib.oracle_kmeans_distortion.restype = ctypes.c_double
        _lib.oracle_centroid_dist.argtypes = [vp, i32, u64, u32, vp, u32, vp]
        _lib.oracle_capacity.argtypes = [u64, u32, u32]
        _lib.oracle_capacity.restype = u64
        _lib.oracle_partition.argtypes = [vp, i32, u64, u32, vp, u32, u32, f32, u32, f32, u64, u32,
                                          vp, vp, vp, vp, vp, vp]
        _lib.oracle_partition.restype = i32
        _lib.oracle_idmap.argtypes = [vp, u64, u32, u32, vp]
        _lib.oracle_idmap.restype = u64
        _lib.oracle_knn.argtypes = [vp, vp, u64, vp, vp, u64, i32, u32, i32, u32, i32, vp, vp]
        _lib.oracle_prune.argtypes = [vp, vp, u64, u32, u32, i32, vp, vp]
        _lib.oracle_reverse.argtypes = [vp, vp, u64, u32, u32, vp, vp]
        _lib.oracle_reverse_lists.argtypes = [vp, vp, u64, u32, vp, vp, vp]
        _lib.oracle_merge.argtypes = [vp, u64, u32, vp, vp, vp, vp, u32, vp, vp]
        _lib.oracle_entry_points.argtypes = [vp, vp, u64, u32, u32, vp, vp]
        _lib.oracle_entry_points.restype = u32
        _lib.oracle_search.argtypes = [vp, i32, u64, u32, vp, u32, u32, vp, u32, u32, u32, i32,
                                       vp, vp, vp]
    return _lib


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p) if a is not None else None


def _data(x):
    x = np.ascontiguousarray(x)
    if x.dtype == np.uint8:
        return x, 0
    return np.ascontiguousarray(x, dtype=np.float32), 1


def kmeans(x, k, seed=42, max_iter=15, spc=256):
    """P0: returns (centroids k x d float32, distortion on the strided sample)."""
    x, dt = _data(x)
    n, d = x.shape
    C = np.zeros((k, d), np.float32)
    dist = ctypes.c_double(0.0)
    st = _load().oracle_kmeans(_p(x), dt, n, d, k, seed, max_iter, spc, _p(C), ctypes.byref(dist))
    if st != 0:
        raise ValueError("oracle_kmeans: bad arguments")
    return C, dist.value


def kmeans_distortion(x, C, spc=256):
    x, dt = _data(x)
    C = np.ascontiguousarray(C, np.float32)
    return _load().oracle_kmeans_distortion(_p(x), dt, x.shape[0], x.shape[1], C.shape[0], spc, _p(C))


def centroid_dist(x, C):
    """P1: n x k float32 squared distances in the fixed fmaf order."""
    x, dt = _data(x)
    C = np.ascontiguousarray(C, np.float32)
    out = np.zeros((x.shape[0], C.shape[0]), np.float32)
    _load().oracle_centroid_dist(_p(x), dt, x.shape[0], x.shape[1], _p(C), C.shape[0], _p(out))
    return out


def capacity(n, k, theta0_ppm=400_000):
    return int(_load().oracle_capacity(n, k, theta0_ppm))


def partition(x, C, omega=2, eps=1.2, theta0_ppm=400_000, alpha=1.0, capacity=0, block_size=65536):
    """P2/P3: returns dict(home n x omega u32, primary_d, sizes, prim, repl, radius)."""
    x, dt = _data(x)
    C = np.ascontiguousarray(C, np.float32)
    n, d = x.shape
    k = C.shape[0]
    home = np.zeros((n, omega), np.uint32)
    pd = np.zeros(n, np.float32)
    sizes = np.zeros(k, np.uint64)
    prim = np.zeros(k, np.uint64)
    repl = np.zeros(k, np.uint64)
    radius = np.zeros(k, np.float32)
    st = _load().oracle_partition(_p(x), dt, n, d, _p(C), k, omega, eps, theta0_ppm, alpha, capacity,
                                  block_size, _p(home), _p(pd), _p(sizes), _p(prim), _p(repl),
                                  _p(radius))
    if st == 4:
        raise RuntimeError("SG_ERR_CAPACITY: every cluster full for a primary")
    return dict(home=home, primary_d=pd, sizes=sizes, prim=prim, repl=repl, radius=radius)


def idmap(home, s):
    home = np.ascontiguousarray(home, np.uint32)
    n, omega = home.shape
    m = _load().oracle_idmap(_p(home), n, omega, s, None)
    out = np.zeros(m, np.uint32)
    _load().oracle_idmap(_p(home), n, omega, s, _p(out))
    return out


def knn(xa, L, xb=None, ida=None, idb=None, self_exclude=True, metric=0):
    """P4: exact top-L.  xb None -> self-join of xa (rows ida)."""
    xa, dt = _data(xa)
    if xb is None:
        xb, idb = xa, ida
    else:
        xb, dt2 = _data(xb)
        assert dt2 == dt
    ida = None if ida is None else np.ascontiguousarray(ida, np.uint32)
    idb = None if idb is None else np.ascontiguousarray(idb, np.uint32)
    ma = xa.shape[0] if ida is None else ida.shape[0]
    mb = xb.shape[0] if idb is None else idb.shape[0]
    ids = np.zeros((ma, L), np.uint32)
    dd = np.zeros((ma, L), np.float32)
    _load().oracle_knn(_p(xa), _p(ida), ma, _p(xb), _p(idb), mb, dt, xa.shape[1], int(self_exclude),
                       L, metric, _p(ids), _p(dd))
    return ids, dd


def prune(knn_ids, knn_d, R, rule=0):
    """P5: rank-based detour-count prune to R (parity unpinned by the paper)."""
    knn_ids = np.ascontiguousarray(knn_ids, np.uint32)
    knn_d = np.ascontiguousarray(knn_d, np.float32)
    m, L = knn_ids.shape
    out = np.zeros((m, R), np.uint32)
    od = np.zeros((m, R), np.float32)
    _load().oracle_prune(_p(knn_ids), _p(knn_d), m, L, R, rule, _p(out), _p(od))
    return out, od


def reverse(pruned, pruned_d, protected=None):
    """P6: reverse-edge insertion, h = floor(R/2) protected forward edges by default."""
    pruned = np.ascontiguousarray(pruned, np.uint32)
    pruned_d = np.ascontiguousarray(pruned_d, np.float32)
    m, R = pruned.shape
    h = R // 2 if protected is None else protected
    out = np.zeros((m, R), np.uint32)
    od = np.zeros((m, R), np.float32)
    _load().oracle_reverse(_p(pruned), _p(pruned_d), m, R, h, _p(out), _p(od))
    return out, od


def reverse_lists(pruned, pruned_d):
    """P6's rev[y] lists (reading R11): sources x in (k, x) order, capped at R.  Returns
    (rev m x R SENT-padded, rev_d carried d(x -> y), counts)."""
    pruned = np.ascontiguousarray(pruned, np.uint32)
    pruned_d = np.ascontiguousarray(pruned_d, np.float32)
    m, R = pruned.shape
    rev = np.zeros((m, R), np.uint32)
    rd = np.zeros((m, R), np.float32)
    rc = np.zeros(m, np.uint32)
    _load().oracle_reverse_lists(_p(pruned), _p(pruned_d), m, R, _p(rev), _p(rd), _p(rc))
    return rev, rd, rc


def merge(home, idmaps, graphs, graphs_d):
    """P7: union + re-prune of the shard graphs into an n x R global graph."""
    home = np.ascontiguousarray(home, np.uint32)
    n, omega = home.shape
    k = len(idmaps)
    R = graphs[0].shape[1]
    idmaps = [np.ascontiguousarray(a, np.uint32) for a in idmaps]
    graphs = [np.ascontiguousarray(a, np.uint32) for a in graphs]
    graphs_d = [np.ascontiguousarray(a, np.float32) for a in graphs_d]
    P = ctypes.c_void_p * k
    sizes = np.array([len(a) for a in idmaps], np.uint64)
    merged = np.zeros((n, R), np.uint32)
    md = np.zeros((n, R), np.float32)
    _load().oracle_merge(_p(home), n, omega, P(*[_p(a) for a in idmaps]), _p(sizes),
                         P(*[_p(a) for a in graphs]), P(*[_p(a) for a in graphs_d]), R, _p(merged),
                         _p(md))
    return merged, md


def entry_points(home, primary_d, sizes):
    home = np.ascontiguousarray(home, np.uint32)
    n, omega = home.shape
    k = len(sizes)
    eps_ = np.zeros(k, np.uint32)
    sizes = np.ascontiguousarray(sizes, np.uint64)
    g = _load().oracle_entry_points(_p(home), _p(np.ascontiguousarray(primary_d, np.float32)), n, omega,
                                    k, _p(sizes), _p(eps_))
    return int(g), eps_


def search(x, graph, entry, queries, topk=10, beam=64, metric=0):
    """P8: greedy beam search; returns (ids nq x topk, dists, distance counts)."""
    x, dt = _data(x)
    q, dq = _data(queries)
    assert dq == dt
    graph = np.ascontiguousarray(graph, np.uint32)
    n, d = x.shape
    R = graph.shape[1]
    nq = q.shape[0]
    ids = np.zeros((nq, topk), np.uint32)
    dd = np.zeros((nq, topk), np.float32)
    nd = np.zeros(nq, np.uint64)
    _load().oracle_search(_p(x), dt, n, d, _p(graph), R, entry, _p(q), nq, topk, beam, metric, _p(ids),
                          _p(dd), _p(nd))
    return ids, dd, nd


def search_shards(x, graph, entries, queries, topk=10, beam=64, metric=0):
    """Split-only search (split-only systems search every shard and merge the
    results; reading R15): P8 from each entry point with its own beam, then per query the
    union of the per-entry top-topk lists ordered by (dist, id), each id once, first topk."""
    per = [search(x, graph, e, queries, topk, beam, metric)[:2] for e in entries]
    nq = per[0][0].shape[0]
    out = np.full((nq, topk), SENT, np.uint32)
    for qi in range(nq):
        cand = {}
        for ids, dd in per:
            for i, dv in zip(ids[qi].tolist(), dd[qi].tolist()):
                if i != SENT:
                    cand[i] = dv
        best = sorted(cand.items(), key=lambda t: (t[1], t[0]))[:topk]
        out[qi, :len(best)] = [i for i, _ in best]
    return out


def recall(ret, gt, k=10):
    """recall@k = |ret[:, :k] & gt[:, :k]| / k averaged over queries."""
    ret = np.asarray(ret)[:, :k]
    gt = np.asarray(gt)[:, :k]
    hits = sum(len(set(r.tolist()) & set(g.tolist())) for r, g in zip(ret, gt))
    return hits / (k * len(gt))
