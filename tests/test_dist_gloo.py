"""World-size-2 tests of the multi-GPU host logic on CPU (gloo backend, 127.0.0.1).

What runs per rank is the product's host code (paper_2605_10135_b200.pipeline): LPT shard
placement and the bootstrap of the library's NCCL communicator (rank 0's unique id shared over
the process group).  The collectives themselves (N1 centroid broadcast, N2 record exchange) run
on that communicator on GPUs; here the merge PROTOCOL of include/scalegann.h is replayed on the
CPU with the oracle's shard graphs and a gloo all-to-all standing in for N2: a row built on a
rank whose primary is owned by another rank travels as a record [g, h, R global ids, R dist
bits] (grouped by destination, ascending g); counts are derived from home[] alone on both sides.
The merged rows each rank ends up owning must equal the single-process oracle merge.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

SENT = 0xFFFFFFFF


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _problem():
    import oracle
    from paper_2605_10135_b200 import datagen
    x = datagen.sift_like(3000, 32, seed=5).numpy()
    k, omega, L, R = 4, 2, 16, 8
    C, _ = oracle.kmeans(x, k)
    part = oracle.partition(x, C, omega=omega, block_size=1024)
    home = part["home"]
    idmaps = [oracle.idmap(home, s) for s in range(k)]
    graphs, graphs_d = [], []
    for s in range(k):
        ki, kd = oracle.knn(x, L, ida=idmaps[s], xb=x, idb=idmaps[s])
        pr, prd = oracle.prune(ki, kd, R)
        g, gd = oracle.reverse(pr, prd)
        graphs.append(g)
        graphs_d.append(gd)
    return x, C, home, idmaps, graphs, graphs_d, R


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        from paper_2605_10135_b200 import pipeline
        x, C, home, idmaps, graphs, graphs_d, R = _problem()
        n, omega = home.shape
        k = len(idmaps)
        W = 2 + 2 * R
        # N1 stand-in: rank 0's centroids reach every rank
        Ct = torch.from_numpy(C.copy()) if rank == 0 else torch.zeros(C.shape, dtype=torch.float32)
        dist.broadcast(Ct, src=0)
        assert np.array_equal(Ct.numpy(), C)
        # shard placement: identical on every rank, deterministic, balanced by m^2
        sizes = [len(a) for a in idmaps]
        owner = pipeline.lpt_owner(sizes, world)
        # pack: rows (h >= 1) of shards owned here whose primary is owned by another rank
        inv = [dict(zip(a.tolist(), range(len(a)))) for a in idmaps]
        per_dest = [[] for _ in range(world)]
        for g in range(n):
            for h in range(1, omega):
                s = int(home[g, h])
                if s == SENT or owner[s] != rank or owner[int(home[g, 0])] == rank:
                    continue
                row = graphs[s][inv[s][g]]
                gid = np.where(row == SENT, SENT, idmaps[s][np.minimum(row, len(idmaps[s]) - 1)]).astype(np.uint32)
                rec = np.concatenate([[g, h], gid, graphs_d[s][inv[s][g]].view(np.uint32)]).astype(np.uint32)
                per_dest[owner[int(home[g, 0])]].append(rec)
        send = [len(r) for r in per_dest]
        sendbuf = torch.from_numpy(np.concatenate([np.stack(r) if r else np.zeros((0, W), np.uint32)
                                                   for r in per_dest]).view(np.int32).reshape(-1).copy())
        # receive counts from home alone (what scalegann_merge_plan computes on the device)
        recv = [0] * world
        for g in range(n):
            if owner[int(home[g, 0])] != rank:
                continue
            for h in range(1, omega):
                s = int(home[g, h])
                if s != SENT and owner[s] != rank:
                    recv[owner[s]] += 1
        recvbuf = torch.empty(max(sum(recv), 1) * W, dtype=torch.int32)
        dist.all_to_all_single(recvbuf[: sum(recv) * W], sendbuf[: sum(send) * W], [c * W for c in recv],
                               [c * W for c in send])
        recs = recvbuf[: sum(recv) * W].numpy().view(np.uint32).reshape(-1, W)
        # union on the owner: local shard rows + received replica rows, through the oracle merge
        lg = [graphs[s].copy() if owner[s] == rank else np.full_like(graphs[s], SENT) for s in range(k)]
        lgd = [graphs_d[s].copy() if owner[s] == rank else np.full_like(graphs_d[s], np.inf) for s in range(k)]
        for rec in recs:
            g, h = int(rec[0]), int(rec[1])
            s = int(home[g, h])
            ids = rec[2:2 + R]
            lg[s][inv[s][g]] = np.array([SENT if v == SENT else inv[s][int(v)] for v in ids], np.uint32)
            lgd[s][inv[s][g]] = rec[2 + R:].view(np.float32)
        merged, _ = oracle.merge(home, idmaps, lg, lgd)
        mine = np.array([owner[int(home[g, 0])] == rank for g in range(n)])
        out[rank] = (mine, merged, owner, send, recv)
    finally:
        dist.destroy_process_group()


def test_distributed_merge_protocol_world2():
    import oracle
    port = _free_port()
    with mp.Manager() as mgr:
        out = mgr.dict()
        mp.spawn(_worker, args=(2, port, out), nprocs=2, join=True)
        res = dict(out)
    x, C, home, idmaps, graphs, graphs_d, R = _problem()
    ref, _ = oracle.merge(home, idmaps, graphs, graphs_d)
    mine0, m0, own0, send0, recv0 = res[0]
    mine1, m1, own1, send1, recv1 = res[1]
    assert own0 == own1                                  # same placement on every rank
    assert np.array_equal(mine0, ~mine1)                 # every global row has exactly one owner
    assert send0[1] == recv1[0] and send1[0] == recv0[1]  # counts agree pairwise
    assert np.array_equal(m0[mine0], ref[mine0])
    assert np.array_equal(m1[mine1], ref[mine1])


def test_lpt_owner_properties():
    from paper_2605_10135_b200.pipeline import lpt_owner
    sizes = [404187, 479168, 434868, 374272, 10, 0]
    for world in (1, 2, 3, 4, 8):
        o = lpt_owner(sizes, world)
        assert o == lpt_owner(sizes, world) and all(0 <= r < world for r in o)
        if world >= 4:   # the four big shards land on four different ranks
            assert len({o[s] for s in range(4)}) == 4
        load = [sum(sizes[s] ** 2 for s in range(len(sizes)) if o[s] == r) for r in range(world)]
        assert max(load) <= max(sizes) ** 2 + min(l for l in load) or world == 1


def _uid_worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2605_10135_b200 import pipeline
        out[rank] = pipeline.share_unique_id(rank, world)
    finally:
        dist.destroy_process_group()


def test_share_unique_id_world2():
    """The library communicator's bootstrap: rank 0's NCCL unique id (scalegann_get_unique_id)
    reaches every rank unchanged over the process group (gloo here; nccl on GPUs)."""
    port = _free_port()
    with mp.Manager() as mgr:
        out = mgr.dict()
        mp.spawn(_uid_worker, args=(2, port, out), nprocs=2, join=True)
        res = dict(out)
    assert len(res[0]) == 128 and res[0] == res[1] and any(res[0])
