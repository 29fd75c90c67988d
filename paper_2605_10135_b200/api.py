"""Thin Python binding of libscalegann.so (include/scalegann.h), same names as the C ABI.

Argument marshalling only: every step of the path runs in the library's CUDA kernels.
torch supplies device memory (tensors, workspaces) and the current CUDA stream.  There is no
CPU fallback: if the extension is missing or a call fails, a ScaleGannError is raised.
"""
from __future__ import annotations

import ctypes
import os

import torch

from . import build as _build

SENT = 0xFFFFFFFF
SG_U8, SG_F32 = 0, 1
SG_L2, SG_IP = 0, 1
PREC_AUTO, PREC_F16_EXACT, PREC_TF32, PREC_TF32X3 = 0, 1, 2, 3
_STATUS = {0: "SG_OK", 1: "SG_ERR_INVALID_ARG", 2: "SG_ERR_UNSUPPORTED", 3: "SG_ERR_CUDA",
           4: "SG_ERR_CAPACITY", 5: "SG_ERR_WORKSPACE", 6: "SG_ERR_TOO_SMALL", 7: "SG_ERR_NCCL"}


class ScaleGannError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{_STATUS.get(status, status)}: {msg}")
        self.status = status


class PartitionParams(ctypes.Structure):
    _fields_ = [("k", ctypes.c_uint32), ("omega", ctypes.c_uint32), ("epsilon", ctypes.c_float),
                ("theta0_ppm", ctypes.c_uint32), ("alpha", ctypes.c_float), ("block_size", ctypes.c_uint32),
                ("capacity", ctypes.c_uint64)]


class BuildParams(ctypes.Structure):
    _fields_ = [("L", ctypes.c_uint32), ("R", ctypes.c_uint32), ("metric", ctypes.c_int32),
                ("precision", ctypes.c_int32), ("prune_rule", ctypes.c_uint32),
                ("protected_edges", ctypes.c_uint32)]


_lib = None
EXPORTS = [
    "scalegann_abi_version", "scalegann_last_error", "scalegann_kmeans_workspace", "scalegann_kmeans",
    "scalegann_partition_workspace", "scalegann_partition", "scalegann_shard_idmap_workspace",
    "scalegann_shard_idmap", "scalegann_entry_points", "scalegann_knn_workspace", "scalegann_knn",
    "scalegann_prune", "scalegann_reverse_workspace", "scalegann_reverse", "scalegann_build_shard_workspace",
    "scalegann_build_shard", "scalegann_optimize_from_knn", "scalegann_get_unique_id", "scalegann_comm_init",
    "scalegann_comm_destroy", "scalegann_comm_rank", "scalegann_broadcast_centroids", "scalegann_exchange_records",
    "scalegann_merge_plan_workspace", "scalegann_merge_plan", "scalegann_merge_init", "scalegann_merge_shard",
    "scalegann_merge_finish", "scalegann_merge_workspace", "scalegann_merge", "scalegann_build_index_host",
    "scalegann_search_workspace",
    "scalegann_search_eval", "scalegann_search_shards_workspace", "scalegann_search_eval_shards", "scalegann_gemm_probe", "scalegann_stats_enable", "scalegann_stats_read", "scalegann_knn_profile",
]


def lib_path() -> str:
    return _build.LIB


def load(build_if_missing: bool = True):
    """Load libscalegann.so (building it with nvcc if it is missing or stale)."""
    global _lib
    if _lib is not None:
        return _lib
    if build_if_missing:
        _build.build()
    if not os.path.exists(_build.LIB):
        raise ImportError(f"libscalegann.so not found at {_build.LIB}; run paper_2605_10135_b200.build")
    L = ctypes.CDLL(_build.LIB)
    vp, u64, u32, i32, f32, sz = (ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_int32,
                                  ctypes.c_float, ctypes.c_size_t)
    psz = ctypes.POINTER(ctypes.c_size_t)
    pu64 = ctypes.POINTER(ctypes.c_uint64)
    pu32 = ctypes.POINTER(ctypes.c_uint32)
    P = ctypes.POINTER
    sig = {
        "scalegann_abi_version": ([], ctypes.c_int),
        "scalegann_last_error": ([], ctypes.c_char_p),
        "scalegann_kmeans_workspace": ([u64, u32, u32, u32, psz], i32),
        "scalegann_kmeans": ([vp, i32, u64, u32, u32, u64, u32, u32, vp, vp, sz, vp], i32),
        "scalegann_partition_workspace": ([u64, u32, P(PartitionParams), psz], i32),
        "scalegann_partition": ([vp, i32, u64, u32, vp, P(PartitionParams), vp, vp, pu64, vp, sz, vp], i32),
        "scalegann_shard_idmap_workspace": ([u64, psz], i32),
        "scalegann_shard_idmap": ([vp, u64, u32, u32, vp, vp, pu64, vp, sz, vp], i32),
        "scalegann_entry_points": ([vp, vp, u64, u32, u32, pu64, pu32, pu32, vp, sz, vp], i32),
        "scalegann_knn_workspace": ([u64, u64, u32, i32, u32, i32, psz], i32),
        "scalegann_knn": ([vp, vp, u64, vp, vp, u64, i32, u32, ctypes.c_int, u32, i32, i32, vp, vp, vp, sz, vp], i32),
        "scalegann_prune": ([vp, vp, u64, u32, u32, u32, vp, vp, vp], i32),
        "scalegann_reverse_workspace": ([u64, u32, psz], i32),
        "scalegann_reverse": ([vp, vp, u64, u32, u32, vp, vp, vp, sz, vp], i32),
        "scalegann_build_shard_workspace": ([u64, u32, i32, P(BuildParams), psz], i32),
        "scalegann_build_shard": ([vp, i32, u64, u32, vp, u64, P(BuildParams), vp, vp, vp, vp, vp, sz, vp], i32),
        "scalegann_optimize_from_knn": ([vp, vp, u64, P(BuildParams), vp, vp, vp, sz, vp], i32),
        "scalegann_get_unique_id": ([ctypes.c_char_p], i32),
        "scalegann_comm_init": ([ctypes.c_int, ctypes.c_int, ctypes.c_char_p, P(vp)], i32),
        "scalegann_comm_destroy": ([vp], i32),
        "scalegann_comm_rank": ([vp, P(ctypes.c_int), P(ctypes.c_int)], i32),
        "scalegann_broadcast_centroids": ([vp, vp, u32, u32, vp], i32),
        "scalegann_exchange_records": ([vp, vp, pu64, vp, pu64, u32, vp], i32),
        "scalegann_merge_plan_workspace": ([u64, psz], i32),
        "scalegann_merge_plan": ([vp, u64, u32, u32, P(i32), ctypes.c_int, ctypes.c_int, vp, vp, pu64, pu64, pu64, vp,
                                  sz, vp], i32),
        "scalegann_merge_init": ([u64, u32, vp, vp, vp], i32),
        "scalegann_merge_shard": ([vp, u64, u32, u32, P(i32), ctypes.c_int, ctypes.c_int, u32, vp, u64, vp, vp, u32,
                                   vp, vp, vp, vp, vp, vp], i32),
        "scalegann_merge_finish": ([u32, u32, vp, vp, u64, vp, vp, vp, sz, vp], i32),
        "scalegann_merge_workspace": ([vp, u64, u32, u32, P(i32), vp, u32, psz, pu64, vp], i32),
        "scalegann_build_index_host": ([vp, vp, i32, u64, u32, P(PartitionParams), P(BuildParams), u64, vp, vp, pu64,
                                        pu32, vp], i32),
        "scalegann_merge": ([vp, vp, u64, u32, u32, P(i32), P(vp), pu64, P(vp), P(vp), u32, vp, vp, pu64, vp, sz,
                             vp], i32),
        "scalegann_search_workspace": ([u64, u32, i32, u32, u32, u32, psz], i32),
        "scalegann_search_eval": ([vp, i32, u64, u32, vp, u32, u32, vp, u32, u32, u32, i32, vp, vp, vp,
                                   P(ctypes.c_double), pu64, vp, sz, vp], i32),
        "scalegann_search_shards_workspace": ([u64, u32, i32, u32, u32, u32, u32, psz], i32),
        "scalegann_search_eval_shards": ([vp, i32, u64, u32, vp, u32, P(u32), u32, vp, u32, u32, u32, i32, vp, vp,
                                          vp, P(ctypes.c_double), pu64, vp, sz, vp], i32),
        "scalegann_gemm_probe": ([vp, u64, vp, u64, i32, u32, i32, vp, vp, sz, vp], i32),
        "scalegann_stats_enable": ([ctypes.c_int], i32),
        "scalegann_knn_profile": ([vp], i32),
        "scalegann_stats_read": ([P(ctypes.c_double), pu64, pu64, ctypes.c_int], i32),
    }
    for name, (args, res) in sig.items():
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = res
    _lib = L
    return L


def _check(st: int):
    if st != 0:
        msg = _lib.scalegann_last_error().decode(errors="replace")
        raise ScaleGannError(st, msg)


def _ptr(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _stream():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def _dtype(x: torch.Tensor) -> int:
    if x.dtype == torch.uint8:
        return SG_U8
    if x.dtype == torch.float32:
        return SG_F32
    raise TypeError(f"vectors must be uint8 or float32, got {x.dtype}")


def _dev(t: torch.Tensor, name: str):
    if not t.is_cuda or not t.is_contiguous():
        raise ValueError(f"{name} must be a contiguous CUDA tensor")


class Workspace:
    """A reusable device scratch buffer (grows on demand)."""

    def __init__(self, device=None):
        self.buf = None
        self.device = device

    def get(self, nbytes: int) -> torch.Tensor:
        nbytes = max(int(nbytes), 256)
        if self.buf is None or self.buf.numel() < nbytes:
            self.buf = None   # release the smaller buffer before the larger one is allocated
            self.buf = torch.empty(nbytes, dtype=torch.uint8, device=self.device or "cuda")
        return self.buf


_WS = {}


def _ws(nbytes: int, ws: Workspace | None):
    if ws is None:
        dev = torch.cuda.current_device()
        ws = _WS.setdefault(dev, Workspace(f"cuda:{dev}"))
    buf = ws.get(nbytes)
    return _ptr(buf), buf.numel()


def _size_q(fn, *args) -> int:
    out = ctypes.c_size_t(0)
    _check(fn(*args, ctypes.byref(out)))
    return out.value


# ----------------------------------------------------------------------------- a1
def scalegann_kmeans(x, k, seed=42, max_iter=15, spc=256, ws=None):
    L = load()
    _dev(x, "x")
    n, d = x.shape
    C = torch.empty(k, d, dtype=torch.float32, device=x.device)
    nb = _size_q(L.scalegann_kmeans_workspace, n, d, k, spc)
    p, nbytes = _ws(nb, ws)
    _check(L.scalegann_kmeans(_ptr(x), _dtype(x), n, d, k, seed, max_iter, spc, _ptr(C), p, nbytes, _stream()))
    return C


# ----------------------------------------------------------------------------- a2-a3
def scalegann_partition(x, centroids, omega=2, epsilon=1.2, theta0_ppm=400_000, alpha=1.0, block_size=65536,
                        capacity=0, ws=None):
    """Returns (home n x omega uint32, primary_d n float32, counts dict of numpy-free python lists)."""
    L = load()
    _dev(x, "x")
    _dev(centroids, "centroids")
    n, d = x.shape
    k = centroids.shape[0]
    prm = PartitionParams(k, omega, epsilon, theta0_ppm, alpha, block_size, capacity)
    home = torch.empty(n, omega, dtype=torch.int32, device=x.device)
    pd = torch.empty(n, dtype=torch.float32, device=x.device)
    counts = (ctypes.c_uint64 * (3 * k))()
    nb = _size_q(L.scalegann_partition_workspace, n, d, ctypes.byref(prm))
    p, nbytes = _ws(nb, ws)
    _check(L.scalegann_partition(_ptr(x), _dtype(x), n, d, _ptr(centroids), ctypes.byref(prm), _ptr(home), _ptr(pd),
                                 counts, p, nbytes, _stream()))
    c = list(counts)
    return home, pd, {"sizes": c[:k], "prim": c[k:2 * k], "repl": c[2 * k:]}


# ----------------------------------------------------------------------------- a4
def scalegann_shard_idmap(home, shard, m=None, inv=None, ws=None):
    """idmap (int32 view of uint32 ids) of `shard`; fills inv (n x omega) if given."""
    L = load()
    _dev(home, "home")
    n, omega = home.shape
    nb = _size_q(L.scalegann_shard_idmap_workspace, n)
    p, nbytes = _ws(nb, ws)
    if m is None:
        mh = ctypes.c_uint64(0)
        _check(L.scalegann_shard_idmap(_ptr(home), n, omega, shard, None, None, ctypes.byref(mh), p, nbytes, _stream()))
        m = mh.value
    idmap = torch.empty(max(m, 1), dtype=torch.int32, device=home.device)
    _check(L.scalegann_shard_idmap(_ptr(home), n, omega, shard, _ptr(idmap), _ptr(inv), None, p, nbytes, _stream()))
    return idmap[:m]


def scalegann_entry_points(home, primary_d, sizes, ws=None):
    L = load()
    n, omega = home.shape
    k = len(sizes)
    sz = (ctypes.c_uint64 * k)(*sizes)
    ent = (ctypes.c_uint32 * k)()
    g = ctypes.c_uint32(0)
    p, nbytes = _ws(64 * 8 + 1024, ws)
    _check(L.scalegann_entry_points(_ptr(home), _ptr(primary_d), n, omega, k, sz, ent, ctypes.byref(g), p, nbytes,
                                    _stream()))
    return g.value, list(ent)


# ----------------------------------------------------------------------------- a5
def scalegann_knn(xa, L_, xb=None, ida=None, idb=None, self_exclude=True, metric=SG_L2, precision=PREC_AUTO,
                  ws=None):
    """Exact top-L: returns (ids ma x L int32 [uint32 bits], dists ma x L float32)."""
    L = load()
    _dev(xa, "xa")
    same = xb is None
    if same:
        xb, idb = xa, ida
    _dev(xb, "xb")
    d = xa.shape[1]
    ma = xa.shape[0] if ida is None else ida.numel()
    mb = xb.shape[0] if idb is None else idb.numel()
    ids = torch.empty(ma, L_, dtype=torch.int32, device=xa.device)
    dist = torch.empty(ma, L_, dtype=torch.float32, device=xa.device)
    nb = _size_q(L.scalegann_knn_workspace, ma, mb, d, _dtype(xa), L_, precision)
    p, nbytes = _ws(nb, ws)
    _check(L.scalegann_knn(_ptr(xa), _ptr(ida), ma, _ptr(xb), _ptr(idb), mb, _dtype(xa), d, int(self_exclude), L_,
                           metric, precision, _ptr(ids), _ptr(dist), p, nbytes, _stream()))
    return ids, dist


def scalegann_gemm_probe(xa, xb, precision=PREC_AUTO, ws=None):
    L = load()
    ma, d = xa.shape
    mb = xb.shape[0]
    out = torch.zeros(ma, mb, dtype=torch.float32, device=xa.device)
    nb = _size_q(L.scalegann_knn_workspace, ma, mb, d, _dtype(xa), 1, precision)
    p, nbytes = _ws(nb, ws)
    _check(L.scalegann_gemm_probe(_ptr(xa), ma, _ptr(xb), mb, _dtype(xa), d, precision, _ptr(out), p, nbytes,
                                  _stream()))
    return out


# ----------------------------------------------------------------------------- a6 / a7
def scalegann_prune(knn_ids, knn_d, R, rule=0):
    L = load()
    m, L_ = knn_ids.shape
    out = torch.empty(m, R, dtype=torch.int32, device=knn_ids.device)
    od = torch.empty(m, R, dtype=torch.float32, device=knn_ids.device)
    _check(L.scalegann_prune(_ptr(knn_ids), _ptr(knn_d), m, L_, R, rule, _ptr(out), _ptr(od), _stream()))
    return out, od


def scalegann_reverse(pruned, pruned_d, protected=None, ws=None):
    L = load()
    m, R = pruned.shape
    h = R // 2 if protected is None else protected
    out = torch.empty(m, R, dtype=torch.int32, device=pruned.device)
    od = torch.empty(m, R, dtype=torch.float32, device=pruned.device)
    nb = _size_q(L.scalegann_reverse_workspace, m, R)
    p, nbytes = _ws(nb, ws)
    _check(L.scalegann_reverse(_ptr(pruned), _ptr(pruned_d), m, R, h, _ptr(out), _ptr(od), p, nbytes, _stream()))
    return out, od


def build_params(L_, R, metric=SG_L2, precision=PREC_AUTO, prune_rule=0, protected_edges=0):
    return BuildParams(L_, R, metric, precision, prune_rule, protected_edges)


def scalegann_build_shard(x, idmap, L_, R, metric=SG_L2, precision=PREC_AUTO, prune_rule=0, protected_edges=0,
                          keep_knn=False, ws=None):
    """gather + exact kNN + prune + reverse for one shard; returns (graph, graph_d[, knn_ids, knn_d])."""
    L = load()
    _dev(x, "x")
    n, d = x.shape
    m = idmap.numel()
    prm = build_params(L_, R, metric, precision, prune_rule, protected_edges)
    g = torch.empty(m, R, dtype=torch.int32, device=x.device)
    gd = torch.empty(m, R, dtype=torch.float32, device=x.device)
    kid = torch.empty(m, L_, dtype=torch.int32, device=x.device) if keep_knn else None
    kd = torch.empty(m, L_, dtype=torch.float32, device=x.device) if keep_knn else None
    nb = _size_q(L.scalegann_build_shard_workspace, m, d, _dtype(x), ctypes.byref(prm))
    p, nbytes = _ws(nb, ws)
    _check(L.scalegann_build_shard(_ptr(x), _dtype(x), n, d, _ptr(idmap), m, ctypes.byref(prm), _ptr(kid), _ptr(kd),
                                   _ptr(g), _ptr(gd), p, nbytes, _stream()))
    return (g, gd, kid, kd) if keep_knn else (g, gd)


def scalegann_optimize_from_knn(knn_ids, knn_d, R, prune_rule=0, protected_edges=0, ws=None):
    L = load()
    m, L_ = knn_ids.shape
    prm = build_params(L_, R, SG_L2, PREC_AUTO, prune_rule, protected_edges)
    g = torch.empty(m, R, dtype=torch.int32, device=knn_ids.device)
    gd = torch.empty(m, R, dtype=torch.float32, device=knn_ids.device)
    nb = _size_q(L.scalegann_build_shard_workspace, m, 1, SG_F32, ctypes.byref(prm))
    p, nbytes = _ws(nb, ws)
    _check(L.scalegann_optimize_from_knn(_ptr(knn_ids), _ptr(knn_d), m, ctypes.byref(prm), _ptr(g), _ptr(gd), p,
                                         nbytes, _stream()))
    return g, gd


# ----------------------------------------------------------------------------- a8
def _ptr_array(ts, k):
    arr = (ctypes.c_void_p * k)()
    for s in range(k):
        arr[s] = ts[s].data_ptr() if ts[s] is not None else None
    return arr


# ----------------------------------------------------------------------------- N1 / N2 communicator
def scalegann_get_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(load().scalegann_get_unique_id(buf))
    return buf.raw


def scalegann_comm_init(rank: int, world: int, uid: bytes):
    """The library's NCCL communicator on the current device (opaque handle)."""
    assert len(uid) == 128
    c = ctypes.c_void_p()
    _check(load().scalegann_comm_init(rank, world, uid, ctypes.byref(c)))
    return c


def scalegann_comm_destroy(comm):
    if comm is not None:
        _check(load().scalegann_comm_destroy(comm))


def scalegann_comm_rank(comm):
    r, w = ctypes.c_int(0), ctypes.c_int(0)
    _check(load().scalegann_comm_rank(comm, ctypes.byref(r), ctypes.byref(w)))
    return r.value, w.value


def scalegann_broadcast_centroids(comm, centroids):
    """N1: rank 0's centroids to every rank, in place."""
    _dev(centroids, "centroids")
    k, d = centroids.shape
    _check(load().scalegann_broadcast_centroids(comm, _ptr(centroids), k, d, _stream()))
    return centroids


def scalegann_exchange_records(comm, sendbuf, send, recv, words):
    """N2: per-peer send/recv of merge records; returns the receive buffer (int32 view)."""
    nrecv = sum(recv)
    recvbuf = torch.empty(max(nrecv, 1) * words, dtype=torch.int32, device=sendbuf.device)
    world = len(send)
    _check(load().scalegann_exchange_records(comm, _ptr(sendbuf), (ctypes.c_uint64 * world)(*send), _ptr(recvbuf),
                                             (ctypes.c_uint64 * world)(*recv), words, _stream()))
    return recvbuf


# ----------------------------------------------------------------------------- a8
def scalegann_merge_plan(home, owner, rank, world, ws=None):
    """Returns (owned_index n int32 [uint32 bits], rec_slot n x omega, send list, recv list, n_owned)."""
    L = load()
    _dev(home, "home")
    n, omega = home.shape
    k = len(owner)
    owned_index = torch.empty(n, dtype=torch.int32, device=home.device)
    rec_slot = torch.empty(n, omega, dtype=torch.int32, device=home.device)
    send = (ctypes.c_uint64 * world)()
    recv = (ctypes.c_uint64 * world)()
    no = ctypes.c_uint64(0)
    nb = _size_q(L.scalegann_merge_plan_workspace, n)
    p, nbytes = _ws(nb, ws)
    _check(L.scalegann_merge_plan(_ptr(home), n, omega, k, (ctypes.c_int32 * k)(*owner), rank, world, _ptr(owned_index),
                                  _ptr(rec_slot), send, recv, ctypes.byref(no), p, nbytes, _stream()))
    return owned_index, rec_slot, list(send), list(recv), no.value


def scalegann_merge_init(n_owned, R, device="cuda"):
    merged = torch.empty(max(n_owned, 1), R, dtype=torch.int32, device=device)[:n_owned]
    merged_d = torch.empty(max(n_owned, 1), R, dtype=torch.float32, device=device)[:n_owned]
    _check(load().scalegann_merge_init(n_owned, R, _ptr(merged), _ptr(merged_d), _stream()))
    return merged, merged_d


def scalegann_merge_shard(home, owner, rank, world, shard, idmap, graph, graph_d, owned_index, rec_slot, merged,
                          merged_d, sendbuf):
    n, omega = home.shape
    k = len(owner)
    m, R = graph.shape
    _check(load().scalegann_merge_shard(_ptr(home), n, omega, k, (ctypes.c_int32 * k)(*owner), rank, world, shard,
                                        _ptr(idmap), m, _ptr(graph), _ptr(graph_d), R, _ptr(owned_index),
                                        _ptr(rec_slot), _ptr(merged), _ptr(merged_d), _ptr(sendbuf), _stream()))


def scalegann_merge_finish(omega, owned_index, recvbuf, n_recv, merged, merged_d, ws=None):
    R = merged.shape[1]
    p, nbytes = _ws(4096, ws)
    _check(load().scalegann_merge_finish(omega, R, _ptr(owned_index), _ptr(recvbuf), n_recv, _ptr(merged),
                                         _ptr(merged_d), p, nbytes, _stream()))


def scalegann_merge(home, idmaps, graphs, graphs_d, owner=None, comm=None, ws=None):
    """One-call collective merge of the shards built on this rank (graphs[s] None elsewhere).
    Returns (merged, merged_d): the rows of the globals whose primary shard is owned here, in
    ascending global id (all n rows at world 1)."""
    L = load()
    n, omega = home.shape
    k = len(idmaps)
    owner = [0] * k if owner is None else owner
    R = next(g for g in graphs if g is not None).shape[1]
    own = (ctypes.c_int32 * k)(*owner)
    nbytes_q = ctypes.c_size_t(0)
    no = ctypes.c_uint64(0)
    _check(L.scalegann_merge_workspace(_ptr(home), n, omega, k, own, comm, R, ctypes.byref(nbytes_q),
                                       ctypes.byref(no), _stream()))
    merged = torch.empty(max(no.value, 1), R, dtype=torch.int32, device=home.device)[:no.value]
    merged_d = torch.empty(max(no.value, 1), R, dtype=torch.float32, device=home.device)[:no.value]
    sizes = (ctypes.c_uint64 * k)(*[0 if a is None else a.numel() for a in idmaps])
    p, nbytes = _ws(nbytes_q.value, ws)
    _check(L.scalegann_merge(comm, _ptr(home), n, omega, k, own, _ptr_array(idmaps, k), sizes, _ptr_array(graphs, k),
                             _ptr_array(graphs_d, k), R, _ptr(merged), _ptr(merged_d), ctypes.byref(no), p, nbytes,
                             _stream()))
    return merged, merged_d


# ----------------------------------------------------------------------------- a1-a8, one call
def scalegann_build_index_host(x_host, merged_host, comm=None, k=4, omega=2, epsilon=1.2, theta0_ppm=400_000,
                               alpha=1.0, block_size=65536, capacity=0, L_=128, R=64, metric=SG_L2,
                               precision=PREC_AUTO, prune_rule=0, protected_edges=0, kmeans_seed=42,
                               merged_d_host=None):
    """Whole build from host buffers: x_host (n x d, CPU, pinned for speed) in, this rank's merged
    rows out into merged_host (CPU, capacity n x R).  Returns (n_owned, global entry)."""
    L = load()
    if x_host.is_cuda or merged_host.is_cuda or not x_host.is_contiguous() or not merged_host.is_contiguous():
        raise ValueError("x_host and merged_host must be contiguous host tensors")
    n, d = x_host.shape
    if merged_host.numel() < n * R:
        raise ValueError("merged_host needs room for n x R ids")
    pp = PartitionParams(k, omega, epsilon, theta0_ppm, alpha, block_size, capacity)
    bp = build_params(L_, R, metric, precision, prune_rule, protected_edges)
    no = ctypes.c_uint64(0)
    ent = ctypes.c_uint32(0)
    _check(L.scalegann_build_index_host(comm, _ptr(x_host), _dtype(x_host), n, d, ctypes.byref(pp), ctypes.byref(bp),
                                        kmeans_seed, _ptr(merged_host), _ptr(merged_d_host), ctypes.byref(no),
                                        ctypes.byref(ent), _stream()))
    return no.value, ent.value


# ----------------------------------------------------------------------------- diagnostics
def scalegann_stats_enable(on=True):
    _check(load().scalegann_stats_enable(int(on)))


def scalegann_stats_read(reset=True):
    """(distance-kernel device ms, distance launches, all kernel launches) since the last reset."""
    ms = ctypes.c_double(0)
    kl = ctypes.c_uint64(0)
    al = ctypes.c_uint64(0)
    _check(load().scalegann_stats_read(ctypes.byref(ms), ctypes.byref(kl), ctypes.byref(al), int(reset)))
    return ms.value, kl.value, al.value


def scalegann_knn_profile(counters=None):
    """Attach (or detach with None) an 80-entry int64 CUDA tensor of per-warp cycle counters."""
    _check(load().scalegann_knn_profile(_ptr(counters)))


# ----------------------------------------------------------------------------- a9
def _search_checks(x, graph, queries):
    _dev(x, "x")
    _dev(graph, "graph")
    _dev(queries, "queries")
    if queries.dtype != x.dtype or queries.shape[1] != x.shape[1]:
        raise ValueError(f"queries must match x in dtype and width ({queries.dtype} {tuple(queries.shape)} vs "
                         f"{x.dtype} {tuple(x.shape)})")


def scalegann_search_eval(x, graph, entry, queries, topk=10, beam=64, metric=SG_L2, gt=None, ws=None,
                          return_ndist=False):
    """Returns (out_ids nq x topk, gt nq x topk, recall[, distance computations])."""
    L = load()
    _search_checks(x, graph, queries)
    n, d = x.shape
    R = graph.shape[1]
    nq = queries.shape[0]
    out = torch.empty(nq, topk, dtype=torch.int32, device=x.device)
    gt_out = None
    if gt is None:
        gt_out = torch.empty(nq, topk, dtype=torch.int32, device=x.device)
    rec = ctypes.c_double(0.0)
    nd = ctypes.c_uint64(0)
    nb = _size_q(L.scalegann_search_workspace, n, d, _dtype(x), nq, topk, beam)
    p, nbytes = _ws(nb, ws)
    _check(L.scalegann_search_eval(_ptr(x), _dtype(x), n, d, _ptr(graph), R, entry, _ptr(queries), nq, topk, beam,
                                   metric, _ptr(gt), _ptr(gt_out), _ptr(out), ctypes.byref(rec), ctypes.byref(nd), p,
                                   nbytes, _stream()))
    res = (out, (gt if gt is not None else gt_out), rec.value)
    return res + (nd.value,) if return_ndist else res


def scalegann_search_eval_shards(x, graph, entries, queries, topk=10, beam=64, metric=SG_L2, gt=None, ws=None,
                                 return_ndist=False):
    """Split-only search: one beam per entry point, per-entry results merged.
    Returns (out_ids nq x topk, gt nq x topk, recall[, distance computations])."""
    L = load()
    _search_checks(x, graph, queries)
    n, d = x.shape
    R = graph.shape[1]
    nq = queries.shape[0]
    ne = len(entries)
    ent = (ctypes.c_uint32 * ne)(*entries)
    out = torch.empty(nq, topk, dtype=torch.int32, device=x.device)
    gt_out = None
    if gt is None:
        gt_out = torch.empty(nq, topk, dtype=torch.int32, device=x.device)
    rec = ctypes.c_double(0.0)
    nd = ctypes.c_uint64(0)
    nb = _size_q(L.scalegann_search_shards_workspace, n, d, _dtype(x), nq, topk, beam, ne)
    p, nbytes = _ws(nb, ws)
    _check(L.scalegann_search_eval_shards(_ptr(x), _dtype(x), n, d, _ptr(graph), R, ent, ne, _ptr(queries), nq, topk,
                                          beam, metric, _ptr(gt), _ptr(gt_out), _ptr(out), ctypes.byref(rec),
                                          ctypes.byref(nd), p, nbytes, _stream()))
    res = (out, (gt if gt is not None else gt_out), rec.value)
    return res + (nd.value,) if return_ndist else res
