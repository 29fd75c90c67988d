"""One pass of the ScaleGANN hot path through the C ABI.

    a1  centroids: scalegann_kmeans on rank 0, N1 scalegann_broadcast_centroids
    a2-a3 partition: scalegann_partition, identical on every rank
    a4-a7 per owned shard: scalegann_shard_idmap + scalegann_build_shard, each shard
        folded into the merged rows (scalegann_merge_shard) and freed before the next one
    a8  merge: N2 scalegann_exchange_records of the rows whose primary is owned elsewhere, then
        scalegann_merge_finish

Shard placement across ranks is LPT on m^2 (the exact kNN costs O(m^2) per shard); shards are
independent builds ("no ... inter-GPU communication").  Both collectives run on the
library's own NCCL communicator (share_unique_id bootstraps it over torch.distributed); they
are the only data exchanged between ranks.
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
    merged: torch.Tensor          # n_owned x R global ids: rows of the globals whose primary shard is owned here
    merged_d: torch.Tensor
    entry: int
    home: torch.Tensor
    primary_d: torch.Tensor
    centroids: torch.Tensor
    sizes: list
    counts: dict
    owner: list
    stage_ms: dict
    owned_index: torch.Tensor | None = None   # row of g in merged (SENT if owned elsewhere)
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


def share_unique_id(rank: int, world: int) -> bytes:
    """Rank 0's 128-byte NCCL unique id to every rank over the torch.distributed process group
    (bootstrap only; works with gloo and nccl)."""
    uid = api.scalegann_get_unique_id() if rank == 0 else bytes(128)
    if world > 1:
        obj = [uid]
        dist.broadcast_object_list(obj, src=0)
        uid = obj[0]
    return uid


def make_comm(rank: int, world: int):
    """The library communicator for this rank (None at world 1)."""
    if world == 1:
        return None
    return api.scalegann_comm_init(rank, world, share_unique_id(rank, world))


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


def build_index(x: torch.Tensor, cfg: BuildConfig, rank: int = 0, world: int = 1, comm=None, timing: bool = False,
                ws: api.Workspace | None = None) -> Index:
    n, d = x.shape
    tm = _Timer(timing)
    # a1 — centroids on rank 0, broadcast (N1)
    tm.mark("a1_kmeans")
    if rank == 0:
        C = api.scalegann_kmeans(x, cfg.k, seed=cfg.kmeans_seed, max_iter=cfg.kmeans_iters, spc=cfg.kmeans_spc, ws=ws)
    else:
        C = torch.empty(cfg.k, d, dtype=torch.float32, device=x.device)
    api.scalegann_broadcast_centroids(comm, C)
    # a2-a3 — partition (identical on every rank)
    tm.mark("a2a3_partition")
    home, pd, counts = api.scalegann_partition(x, C, omega=cfg.omega, epsilon=cfg.epsilon,
                                               theta0_ppm=cfg.theta0_ppm, alpha=cfg.alpha,
                                               block_size=cfg.block_size, capacity=cfg.capacity, ws=ws)
    sizes = counts["sizes"]
    owner = lpt_owner(sizes, world)
    R, W = cfg.R, 2 + 2 * cfg.R
    owned_index, rec_slot, send, recv, n_owned = api.scalegann_merge_plan(home, owner, rank, world, ws=ws)
    merged, merged_d = api.scalegann_merge_init(n_owned, R, device=x.device)
    sendbuf = torch.empty(max(sum(send), 1) * W, dtype=torch.int32, device=x.device)
    # a4-a7 — owned shards, each folded into the merged rows and freed
    tm.mark("a4a7_build")
    for s in range(cfg.k):
        if owner[s] != rank or sizes[s] == 0:
            continue
        idmap = api.scalegann_shard_idmap(home, s, m=sizes[s], ws=ws)
        g, gd = api.scalegann_build_shard(x, idmap, cfg.L, cfg.R, metric=cfg.metric, precision=cfg.precision,
                                          prune_rule=cfg.prune_rule, protected_edges=cfg.protected_edges, ws=ws)
        api.scalegann_merge_shard(home, owner, rank, world, s, idmap, g, gd, owned_index, rec_slot, merged, merged_d,
                                  sendbuf)
        del g, gd, idmap
    # a8 — rows whose primary lives elsewhere travel to its owner (N2), then fold
    tm.mark("a8_merge")
    if world > 1:
        recvbuf = api.scalegann_exchange_records(comm, sendbuf, send, recv, W)
        api.scalegann_merge_finish(cfg.omega, owned_index, recvbuf, sum(recv), merged, merged_d, ws=ws)
    tm.mark("end")
    entry, _ = api.scalegann_entry_points(home, pd, sizes, ws=ws)
    return Index(merged, merged_d, entry, home, pd, C, sizes, counts, owner, tm.result(), owned_index=owned_index)


def gather_merged(index: "Index", rank: int, world: int) -> torch.Tensor | None:
    """The full n x R merged graph on rank 0 (evaluation only): every rank's owned rows placed at
    their global ids (torch.distributed gather).  Other ranks return None."""
    n = index.home.shape[0]
    if world == 1:
        return index.merged
    R = index.merged.shape[1]
    full = torch.full((n, R), -1, dtype=torch.int32, device=index.merged.device)
    own = owned_rows(index, rank)
    full[own] = index.merged
    dist.all_reduce(full, op=dist.ReduceOp.MAX)   # rows owned elsewhere are -1 here
    return full if rank == 0 else None


def owned_rows(index: Index, rank: int) -> torch.Tensor:
    """Boolean mask of the global ids whose merged row lives on `rank` (primary shard owner)."""
    own = torch.tensor(index.owner, dtype=torch.int64, device=index.home.device)
    return own[index.home[:, 0].long()] == rank
