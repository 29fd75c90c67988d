"""Helper for tests/test_gpu_multi.py, run under torchrun (one rank per GPU, NCCL): the pipeline
with the library's communicator (N1 centroid broadcast, N2 record exchange) on `world` ranks.
Every rank's owned merged rows, reassembled on rank 0, must equal the world = 1 build of the same
data byte for byte (ids and distances), and rank 0 writes the verdict as JSON to argv[1]."""
import json
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    out = sys.argv[1]
    n, k = int(sys.argv[2]), int(sys.argv[3])
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    from paper_2605_10135_b200 import api, datagen
    from paper_2605_10135_b200.pipeline import BuildConfig, build_index, make_comm
    api.load()
    comm = make_comm(rank, world)
    x = datagen.sift_like(n, 128, seed=77, device="cuda")
    cfg = BuildConfig(k=k, L=64, R=32)
    idx = build_index(x, cfg, rank, world, comm)
    torch.cuda.synchronize()
    own = torch.tensor(idx.owner, device="cuda")[idx.home[:, 0].long()] == rank
    full = torch.full((n, cfg.R), -1, dtype=torch.int32, device="cuda")
    full_d = torch.full((n, cfg.R), -1.0, dtype=torch.float32, device="cuda")
    full[own], full_d[own] = idx.merged, idx.merged_d
    dist.all_reduce(full, op=dist.ReduceOp.MAX)
    dist.all_reduce(full_d, op=dist.ReduceOp.MAX)
    if rank == 0:
        ref = build_index(x, cfg)   # world 1, no communicator
        torch.cuda.synchronize()
        res = {"world": world, "n": n, "k": k, "owner": idx.owner, "n_owned_rank0": int(idx.merged.shape[0]),
               "ids_equal": bool(torch.equal(full, ref.merged)), "dists_equal": bool(torch.equal(full_d, ref.merged_d)),
               "home_equal": bool(torch.equal(idx.home, ref.home)), "entry_equal": idx.entry == ref.entry}
        with open(out, "w") as f:
            json.dump(res, f)
    dist.barrier()
    api.scalegann_comm_destroy(comm)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
