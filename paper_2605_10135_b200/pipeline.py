"""One pass of the ScaleGANN hot path through the C ABI.

    a1  centroids: scalegann_kmeans on rank 0, NCCL broadcast to every rank
    a2-a3 partition: scalegann_partition, identical on every rank
    a4-a7 per owned shard: scalegann_shard_idmap + scalegann_build_shard
    a8  merge: scalegann_merge_pack -> NCCL all-to-all over NVLink -> scalegann_merge_union
        (P:139); single process: scalegann_merge

Shard placement across ranks is LPT on m^2 (the exact kNN costs O(m^2) per shard); shards are
independent builds ("no ... inter-GPU communication").  torch.distributed provides the
process group; the only collectives are the centroid broadcast and the merge all-to-all.
"""
from __future__ import annotations

import dataclasses
import time

import torch
import torch.distributed as dist

from . import api


@dataclasses.dataclass
class BuildConfig:
    k: int
    omega: int = 2
    epsilon: float = 1.2
    theta0_ppm: int = 400_000
    alpha: float = 1.0
    block_size: int = 65536
    capacity: int = 0
    L: int = 128
    R: int = 64
    metric: int = api.SG_L2
    precision: int = api.PREC_AUTO
    prune_rule: int = 0
    protected_edges: int = 0
    kmeans_seed: int = 42
    kmeans_iters: int = 15
    kmeans_spc: int = 256


@dataclasses.dataclass
class Index:
    merged: torch.Tensor          # n x R global ids (rows owned by this rank filled)
    merged_d: torch.Tensor
    entry: int
    home: torch.Tensor
    primary_d: torch.Tensor
    centroids: torch.Tensor
    sizes: list
    counts: dict
    owner: list
    stage_ms: dict
    launches: int = 0


def lpt_owner(sizes, world):
    """Longest-processing-time placement of shards on ranks by m^2 (ties -> lower shard/rank)."""
    order = sorted(range(len(sizes)), key=lambda s: (-(sizes[s] ** 2), s))
    load = [0] * world
    owner = [0] * len(sizes)
    for s in order:
        r = min(range(world), key=lambda q: (load[q], q))
        owner[s] = r
        load[r] += sizes[s] ** 2
    return owner


def broadcast_centroids(C: torch.Tensor, world: int) -> torch.Tensor:
    """N1: rank 0's k x d centroids to every rank (in place; NCCL over NVLink on GPUs)."""
    if world > 1:
        dist.broadcast(C, src=0)
    return C


def exchange_records(sendbuf: torch.Tensor, send: list, recv: list, W: int) -> torch.Tensor:
    """N2: all-to-all of the merge records (W int32 words each).  `send[r]` / `recv[r]` count the
    records this rank sends to / receives from rank r (both known locally from `home`, so no count
    exchange is needed); records arrive grouped by source rank, in rank order."""
    nrecv = sum(recv)
    recvbuf = torch.empty(max(nrecv, 1) * W, dtype=torch.int32, device=sendbuf.device)
    dist.all_to_all_single(recvbuf[: nrecv * W], sendbuf[: sum(send) * W], [c * W for c in recv],
                           [c * W for c in send])
    return recvbuf


def distribute_dataset(x_local: torch.Tensor, n: int, rank: int, world: int) -> torch.Tensor:
    """Every rank holds the full dataset (the partition runs identically everywhere),
    but only its contiguous 1/world slice crosses PCIe: the slices are all-gathered over NVLink.
    `x_local` is this rank's rows [rank*n/world, (rank+1)*n/world) on the device."""
    if world == 1:
        return x_local
    assert n % world == 0, "n must be a multiple of the world size"
    full = torch.empty((n,) + tuple(x_local.shape[1:]), dtype=x_local.dtype, device=x_local.device)
    dist.all_gather_into_tensor(full, x_local.contiguous())
    return full


class _Timer:
    def __init__(self, on: bool):
        self.on = on
        self.ev = []

    def mark(self, name):
        if self.on:
            e = torch.cuda.Event(enable_timing=True)
            e.record()
            self.ev.append((name, e))

    def result(self):
        if not self.on or len(self.ev) < 2:
            return {}
        torch.cuda.synchronize()
        out = {}
        for (n0, e0), (_, e1) in zip(self.ev, self.ev[1:]):
            out[n0] = out.get(n0, 0.0) + e0.elapsed_time(e1)
        return out


def build_index(x: torch.Tensor, cfg: BuildConfig, rank: int = 0, world: int = 1, timing: bool = False,
                ws: api.Workspace | None = None) -> Index:
    n, d = x.shape
    tm = _Timer(timing)
    # a1 — centroids on rank 0, broadcast (N1)
    tm.mark("a1_kmeans")
    if rank == 0:
        C = api.scalegann_kmeans(x, cfg.k, seed=cfg.kmeans_seed, max_iter=cfg.kmeans_iters, spc=cfg.kmeans_spc, ws=ws)
    else:
        C = torch.empty(cfg.k, d, dtype=torch.float32, device=x.device)
    broadcast_centroids(C, world)
    # a2-a3 — partition (identical on every rank)
    tm.mark("a2a3_partition")
    home, pd, counts = api.scalegann_partition(x, C, omega=cfg.omega, epsilon=cfg.epsilon,
                                               theta0_ppm=cfg.theta0_ppm, alpha=cfg.alpha,
                                               block_size=cfg.block_size, capacity=cfg.capacity, ws=ws)
    sizes = counts["sizes"]
    owner = lpt_owner(sizes, world)
    inv = torch.full((n, cfg.omega), -1, dtype=torch.int32, device=x.device)
    idmaps, graphs, graphs_d = [None] * cfg.k, [None] * cfg.k, [None] * cfg.k
    # a4-a7 — owned shards
    tm.mark("a4a7_build")
    for s in range(cfg.k):
        if owner[s] != rank or sizes[s] == 0:
            continue
        idmaps[s] = api.scalegann_shard_idmap(home, s, m=sizes[s], inv=inv, ws=ws)
        graphs[s], graphs_d[s] = api.scalegann_build_shard(x, idmaps[s], cfg.L, cfg.R, metric=cfg.metric,
                                                           precision=cfg.precision, prune_rule=cfg.prune_rule,
                                                           protected_edges=cfg.protected_edges, ws=ws)
    # a8 — merge
    tm.mark("a8_merge")
    if world == 1:
        merged, merged_d = api.scalegann_merge(home, inv, idmaps, graphs, graphs_d, ws=ws)
    else:
        R = cfg.R
        W = 2 + 2 * R
        send, recv = api.scalegann_merge_counts(home, cfg.k, owner, rank, world, ws=ws)
        any_graph = next((g for g in graphs if g is not None), None)
        if any_graph is None:   # a rank without shards still takes part in the exchange
            graphs = [torch.empty(0, R, dtype=torch.int32, device=x.device) if s == 0 else None
                      for s in range(cfg.k)]
        sendbuf = api.scalegann_merge_pack(home, inv, owner, rank, world, idmaps, graphs, graphs_d, sum(send), ws=ws)
        recvbuf = exchange_records(sendbuf, send, recv, W)
        merged, merged_d = api.scalegann_merge_union(home, inv, owner, rank, idmaps, graphs, graphs_d, recvbuf,
                                                     sum(recv), ws=ws)
    tm.mark("end")
    entry, _ = api.scalegann_entry_points(home, pd, sizes, ws=ws)
    return Index(merged, merged_d, entry, home, pd, C, sizes, counts, owner, tm.result())


def owned_rows(index: Index, rank: int) -> torch.Tensor:
    """Boolean mask of the global ids whose merged row lives on `rank` (primary shard owner)."""
    own = torch.tensor(index.owner, dtype=torch.int64, device=index.home.device)
    return own[index.home[:, 0].long()] == rank
