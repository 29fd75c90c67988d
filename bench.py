#!/usr/bin/env python
"""bench.py — ScaleGANN divide-and-merge index build (arxiv 2605.10135) on B200.

One step = one pass of the whole hot path over one synthetic
dataset resident in HBM: k-means centroids + NCCL broadcast, overlapping partition, per-shard
exact kNN (tcgen05) + detour prune + reverse edges, cross-shard merge (+ NCCL all-to-all).

Workload (weak scaling): N GPUs build an N x 1M x 128 SIFT-shaped float32 dataset split into
4N shards (replication omega=2, R=64, L=128) — at N=1 exactly BASELINE.json configs[1]
("SIFT1M-shaped 1Mx128 fp32, 4 shards, replication 2, degree 64 on 1 B200"); every rank owns
4 shards of ~C1 size.  Metric: index-build vectors/s (whole job), plus the distance kernel's
tensor roofline fraction and recall@10 (untimed evaluation).

    python bench.py [--gpus N --steps K --warmup W]            # our CUDA path
    python bench.py --impl reference                           # the CPU oracle (bounded sample)
    torchrun --nproc-per-node N bench.py --gpus N ...          # N > 1 (one rank per GPU, NCCL)
"""
from __future__ import annotations

import argparse
import json
import os

os.environ.setdefault("PYTORCH_CUDA_ALLOC_CONF", "expandable_segments:True")   # big configs: no fragmentation
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "index build vectors/sec"
UNIT = "vectors/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C1", choices=["C1", "C2", "C3", "C4"],
                    help="C1: BASELINE configs[1] weak-scaled (1M x 128 and 4 shards per GPU, the driver's line); "
                         "C2/C3/C4: the fixed 8-shard workloads of SURVEY 8(d) on any number of GPUs")
    ap.add_argument("--n-per-gpu", type=int, default=1_000_000)
    ap.add_argument("--n", type=int, default=0, help="C2-C4: override the dataset size (reduced runs)")
    ap.add_argument("--shards-per-gpu", type=int, default=4)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e", action="store_true", help="C2-C4: also time the host-buffer e2e leg")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-recall", action="store_true")
    ap.add_argument("--no-stages", action="store_true", help="skip the extra untimed step of the stage breakdown")
    ap.add_argument("--no-parity", action="store_true", help="skip the oracle parity check at bench size")
    ap.add_argument("--profile-steps", action="store_true", help="minimal run for ncu (no e2e/cpu/recall)")
    return ap.parse_args()


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, dev_index: int):
        self.dev = dev_index
        self.lines = []
        self.proc = None
        self.t = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                                          "-lms", "200", "-i", str(self.dev)], stdout=subprocess.PIPE,
                                         stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.t.join(timeout=2)
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[1]))
                mx = float(parts[2])
            except ValueError:
                continue
            for nm, v in zip(names, parts[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def oracle_sample_run(x_np, C_np, k, omega, L, sample_rows, home_np=None):
    """One bounded oracle step: full partition (P2/P3) + exact kNN (P4) for `sample_rows` rows
    of every shard against the whole shard, extrapolated to every row.  Returns
    (extrapolated seconds for the full workload, measured seconds, description)."""
    import numpy as np
    import oracle
    t0 = time.perf_counter()
    r = oracle.partition(x_np, C_np, omega=omega)
    t_part = time.perf_counter() - t0
    t_knn_ex, t_knn = 0.0, 0.0
    for s in range(k):
        im = oracle.idmap(r["home"], s)
        m = len(im)
        if m < 2:
            continue
        rows = im[np.linspace(0, m - 1, num=min(sample_rows, m)).astype(np.int64)]
        t1 = time.perf_counter()
        oracle.knn(x_np, L, ida=rows, xb=x_np, idb=im, self_exclude=False)
        dt = time.perf_counter() - t1
        t_knn += dt
        t_knn_ex += dt * m / len(rows)
    desc = (f"full oracle partition of {x_np.shape[0]} vectors + exact kNN of {sample_rows} rows per shard "
            f"against the whole shard ({k} shards), extrapolated x m/{sample_rows}; prune/reverse/merge "
            f"(O(m L^2), <2% of the oracle's kNN work) not timed")
    return t_part + t_knn_ex, t_part + t_knn, desc


def oracle_rows_exact(oracle, x_np, rows, idb, L):
    """P4 top-L of shard rows `rows` (local ids into idb) against the whole shard, self excluded:
    the oracle's top L+1 with the self column included, minus self (if self is not among them,
    >= L+1 exact duplicates with lower ids precede it and the first L are the answer)."""
    import numpy as np
    ids, dd = oracle.knn(x_np, L + 1, ida=idb[rows].astype(np.uint32), xb=x_np, idb=idb, self_exclude=False)
    out_i = np.zeros((len(rows), L), np.uint32)
    out_d = np.zeros((len(rows), L), np.float32)
    for t, r in enumerate(rows):
        keep = ids[t] != r
        if keep.all():
            keep[-1] = False
        out_i[t], out_d[t] = ids[t][keep], dd[t][keep]
    return out_i, out_d


def scale_parity(x, idx, cfg, sample_rows=2000, seed=5):
    """Parity at the bench's own size (after the timed region, in the oracle leg):
      * partition: the oracle's home[] from the library's centroids equals the GPU's, bit for bit;
      * kNN: `sample_rows` rows of the largest shard (first rows, last rows = ragged tail, random)
        have exactly the oracle's P4 top-L (ids and dists);
      * prune + reverse + merge: the oracle fed the GPU's kNN lists of every shard rebuilds the
        merged graph, which must equal the GPU's merged graph byte for byte.
    Returns a dict for the bench line."""
    import numpy as np
    import oracle
    from paper_2605_10135_b200 import api
    oracle.build()
    t0 = time.perf_counter()
    x_np = x.cpu().numpy()
    r = oracle.partition(x_np, idx.centroids.cpu().numpy(), omega=cfg.omega, eps=cfg.epsilon,
                         theta0_ppm=cfg.theta0_ppm, alpha=cfg.alpha, block_size=cfg.block_size)
    home_gpu = idx.home.cpu().numpy().view(np.uint32)
    home_ok = bool(np.array_equal(home_gpu, r["home"]))
    big = max(range(cfg.k), key=lambda s: (idx.sizes[s], -s))
    idm, gs, gds = [], [], []
    knn_rows_ok = knn_rows = 0
    for s in range(cfg.k):
        im = oracle.idmap(r["home"], s)
        im_d = torch_from(im, x.device)
        g, gd, kid, kd = api.scalegann_build_shard(x, im_d, cfg.L, cfg.R, keep_knn=True)
        kid_h = kid.cpu().numpy().view(np.uint32)
        kd_h = kd.cpu().numpy()
        del g, gd, kid, kd
        if s == big:
            m = len(im)
            rng = np.random.default_rng(seed)
            rows = sorted(set(range(min(m, 200))) | set(range(max(0, m - 300), m)) |
                          set(rng.choice(m, size=min(m, max(0, sample_rows - 500)), replace=False).tolist()))
            rows = np.array(rows, np.int64)
            oi, od = oracle_rows_exact(oracle, x_np, rows, im, cfg.L)
            same = (kid_h[rows] == oi).all(1) & (kd_h[rows] == od).all(1)
            knn_rows, knn_rows_ok = len(rows), int(same.sum())
        p, pd = oracle.prune(kid_h, kd_h, cfg.R, rule=cfg.prune_rule)
        f, fd = oracle.reverse(p, pd, protected=cfg.protected_edges or None)
        idm.append(im), gs.append(f), gds.append(fd)
    om, omd = oracle.merge(r["home"], idm, gs, gds)
    merged = idx.merged.cpu().numpy().view(np.uint32)
    merged_ok = bool(np.array_equal(merged, om) and np.array_equal(idx.merged_d.cpu().numpy(), omd))
    return {"home_identical": home_ok,
            "knn_sampled_rows": knn_rows, "knn_rows_identical": knn_rows_ok,
            "knn_sample": f"largest shard ({idx.sizes[big]} rows): first 200, last 300, "
                          f"{max(0, sample_rows - 500)} random rows vs the oracle's exact P4 top-{cfg.L}",
            "replay_merged_identical": merged_ok,
            "replay": "oracle prune + reverse + merge fed the GPU kNN lists of every shard vs the GPU merged graph",
            "seconds": time.perf_counter() - t0}


def torch_from(a, device):
    import numpy as np
    import torch
    return torch.from_numpy(np.ascontiguousarray(a).view(np.int32)).to(device)


def run_reference(args):
    """--impl reference: the CPU oracle as it stands on the host cores (rank 0 only)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import numpy as np
    import oracle
    from paper_2605_10135_b200 import datagen
    oracle.build()
    n = args.n_per_gpu * args.gpus
    k = args.shards_per_gpu * args.gpus
    x = datagen.sift_like(n, 128).numpy()
    C, _ = oracle.kmeans(x, k)
    sample = 8
    times = []
    for it in range(args.warmup + args.steps):
        ext, meas, desc = oracle_sample_run(x, C, k, 2, 128, sample)
        if it >= args.warmup:
            times.append(ext)
    t = statistics.mean(times)
    value = n / t
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t * 1000, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "int64/f64", "data": "synthetic",
            "config": {"workload": f"C1 SIFT-shaped {n}x128 f32 (weak: {args.n_per_gpu} per GPU), {k} shards",
                       "n": n, "d": 128, "k": k, "omega": 2, "L": 128, "R": 64},
            "impl": "reference",
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores(), "kind": "oracle", "sample": desc},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    emit(line)


_OUT_FD = None


def emit(line: dict):
    """The one JSON line on the real stdout; everything else (NCCL's version banner, native
    prints) was redirected to stderr by main()."""
    fd = _OUT_FD if _OUT_FD is not None else 1
    os.write(fd, (json.dumps(line) + "\n").encode())


CONFIGS = {
    # name: (kind, n or None = n_per_gpu * world, d, shards or None = shards_per_gpu * world, scaling)
    "C1": ("sift", None, 128, None, "weak"),
    "C2": ("deep", 10_000_000, 96, 8, "strong"),
    "C3": ("text", 5_000_000, 768, 8, "strong"),
    "C4": ("sift_u8", 100_000_000, 128, 8, "strong"),
}


def main():
    global _OUT_FD
    args = parse()
    sys.stdout.flush()
    _OUT_FD = os.dup(1)
    os.dup2(2, 1)
    if args.impl == "reference":
        run_reference(args)
        return
    import torch
    import torch.distributed as dist
    from paper_2605_10135_b200 import api, datagen
    from paper_2605_10135_b200.pipeline import BuildConfig, build_index, gather_merged, make_comm

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    api.load()
    comm = make_comm(rank, world)   # the library's NCCL communicator: N1 + N2 of the path
    if args.profile_steps:
        args.no_e2e = args.no_cpu_baseline = args.no_recall = True

    kind, n_fix, d, k_fix, scaling = CONFIGS[args.config]
    n = (args.n or n_fix) if n_fix else args.n_per_gpu * world
    k = k_fix if k_fix else args.shards_per_gpu * world
    if args.config != "C1":   # big workloads: the oracle leg and the pinned-host e2e copy off unless asked
        args.no_cpu_baseline = True
        args.no_e2e = args.no_e2e or not args.e2e
    cfg = BuildConfig(k=k, omega=2, L=128, R=64)
    x = datagen._make(kind, n, d, datagen.DATA_SEED, "cuda")
    torch.cuda.synchronize()
    elem = x.element_size()

    def barrier():
        if world > 1:
            dist.barrier()

    def step(inp):
        return build_index(inp, cfg, rank, world, comm)

    idx = None
    for _ in range(args.warmup):
        idx = None   # one index alive at a time (C4 at N = 1: 51 GB of merged rows each)
        idx = step(x)
    torch.cuda.synchronize()
    barrier()

    # ---------------- timed region: inputs resident in HBM (larger than the 126 MB L2 per rank)
    api.scalegann_stats_read(reset=True)
    api.scalegann_stats_enable(True)
    clk = ClockSampler(local)
    clk.start()
    barrier()
    torch.cuda.synchronize()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record()
    for _ in range(args.steps):
        idx = None
        idx = step(x)
    t1.record()
    torch.cuda.synchronize()
    barrier()
    clocks = clk.stop()
    api.scalegann_stats_enable(False)
    knn_ms, knn_launches, launches = api.scalegann_stats_read(reset=True)
    ms = t0.elapsed_time(t1)
    if world > 1:
        tt = torch.tensor([ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = float(tt.item())
    value = n * args.steps / (ms / 1000.0)

    # ---------------- roofline of the dominant kernel (distance tiles, tcgen05)
    owned = [s for s in range(k) if idx.owner[s] == rank]
    alg_flops_step = sum(2.0 * idx.sizes[s] ** 2 * d for s in owned)
    peaks, src = load_peaks()
    prec_is_f16 = kind in ("sift", "sift_u8")   # integer data -> F16_EXACT (AUTO); float -> 3xTF32 (AUTO)
    peak = peaks.get("bf16_tflops_sustained", peaks.get("bf16_tflops")) * (1.0 if prec_is_f16 else 0.5)
    achieved = alg_flops_step * args.steps / (knn_ms / 1000.0) / 1e12 if knn_ms > 0 else None
    traffic, pipe_pct, prof_src = None, None, None
    tp = os.path.join(ROOT, "profiles", "knn_dram_bytes.json")
    if os.path.exists(tp) and args.config == "C1":
        try:
            prof = json.load(open(tp))
            traffic = prof.get("dram_bytes_per_launch")
            pipe_pct = prof.get("tensor_pipe_active_pct")
            prof_src = prof.get("source")
        except Exception:
            traffic = None
    roofline = {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                "frac": (achieved / peak) if achieved else None, "traffic": traffic,
                "ncu_tensor_pipe_active_pct": pipe_pct, "ncu_source": prof_src,
                "kernel": "knn_tc_kernel (tcgen05.mma kind::%s, fp32 accumulate)" % ("f16" if prec_is_f16 else "tf32"),
                "peak_source": f"{src} bf16 dense sustained" + (" (f16 = bf16 rate)" if prec_is_f16 else " x 0.5 (tf32)"),
                "tensor_work_per_algorithmic_flop": 1 if prec_is_f16 else 3,
                "per_unit": f"2*d flops per (row, column) pair; m_s^2 pairs per shard launch (d = {d})",
                "knn_ms_per_step": knn_ms / args.steps, "knn_launches": knn_launches,
                "knn_share_of_step": (knn_ms / args.steps) / (ms / args.steps)}

    # ---------------- e2e through the C ABI with HOST buffers (scalegann_build_index_host: the
    # dataset copied to the device, a1-a8, the owned merged rows copied back, in one call per step)
    e2e = None
    if not args.no_e2e:
        xh = x.cpu().pin_memory()
        outh = torch.empty(n * cfg.R, dtype=torch.int32, pin_memory=True)
        h2d = xh.numel() * elem * world
        kw = dict(k=cfg.k, omega=cfg.omega, epsilon=cfg.epsilon, theta0_ppm=cfg.theta0_ppm, alpha=cfg.alpha,
                  block_size=cfg.block_size, L_=cfg.L, R=cfg.R, kmeans_seed=cfg.kmeans_seed)
        idx = None   # the device-timed index is not needed any more (C4 memory)
        api.scalegann_build_index_host(xh, outh, comm, **kw)   # warm-up (stream-ordered pool)
        barrier()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.steps):
            n_owned, _ = api.scalegann_build_index_host(xh, outh, comm, **kw)
        e1.record()
        torch.cuda.synchronize()
        barrier()
        ems = e0.elapsed_time(e1)
        d2h_local = n_owned * cfg.R * 4
        d2h = d2h_local
        if world > 1:
            tt = torch.tensor([ems, float(d2h_local)], dtype=torch.float64, device="cuda")
            t_max = tt.clone()
            dist.all_reduce(t_max, op=dist.ReduceOp.MAX)
            dist.all_reduce(tt, op=dist.ReduceOp.SUM)
            ems, d2h = float(t_max[0].item()), int(tt[1].item())
        e2e = {"value": n * args.steps / (ems / 1000.0), "unit": UNIT, "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": d2h, "ms_per_step": ems / args.steps,
               "api": "scalegann_build_index_host (one C-ABI call per step, host buffers in and out)",
               "note": "whole-job bytes: the full dataset to every rank, each rank's owned merged rows back"}
        del xh, outh
        idx = step(x)   # the device index again, for the legs below

    # ---------------- per-stage breakdown from one extra (untimed) step
    stage_ms = None if args.no_stages else build_index(x, cfg, rank, world, comm, timing=True).stage_ms

    # ---------------- recall@10 of the merged graph (untimed evaluation, a9)
    recall = None
    if not args.no_recall:
        full = gather_merged(idx, rank, world)
        if rank == 0:
            nq = 10_000 if args.config == "C1" else 1000
            q = datagen._make(kind, nq, d, datagen.DATA_SEED + datagen.QUERY_SEED_OFFSET, "cuda")
            recall = {}
            gt = None
            for beam in (32, 64, 128):
                _, gt, r = api.scalegann_search_eval(x, full, idx.entry, q, topk=10, beam=beam, gt=gt)
                recall[f"beam{beam}"] = r
        del full

    # ---------------- CPU oracle baseline + parity at bench size (rank 0, N=1 only)
    cpu = None
    parity = None
    if not args.no_cpu_baseline and world == 1 and rank == 0:
        import oracle
        oracle.build()
        sample = 8
        ext, meas, desc = oracle_sample_run(x.cpu().numpy(), idx.centroids.cpu().numpy(), k, 2, 128, sample)
        cpu = {"value": n / ext, "unit": UNIT, "cores": cores(), "kind": "oracle", "sample": desc,
               "measured_s": meas, "extrapolated_s": ext}
        if not args.no_parity:
            parity = scale_parity(x, idx, cfg)

    if rank == 0:
        wl = {"C1": f"C1 SIFT-shaped {n}x128 f32 integer-valued (weak: {n // world} per GPU)",
              "C2": f"C2 DEEP-shaped {n}x96 f32 L2-normalised, {k} shards on {world} GPU(s)",
              "C3": f"C3 text-embedding-shaped {n}x768 f32, {k} shards on {world} GPU(s)",
              "C4": f"C4 BIGANN-shaped {n}x128 u8, {k} shards on {world} GPU(s)"}[args.config]
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": scaling,
            "vs_baseline": None, "dtype": "f16" if prec_is_f16 else "tf32x3", "data": "synthetic",
            "config": {"workload": wl, "n": n, "d": d, "k": k, "omega": 2, "epsilon": 1.2, "L": 128, "R": 64,
                       "precision": ("F16_EXACT operands, fp32 accumulate (exact for this integer data)"
                                     if prec_is_f16 else "3xTF32 operands (AUTO: hi/lo split, ~fp32 products), fp32 accumulate"),
                       "shard_sizes": idx.sizes, "replicas": sum(idx.counts["repl"]),
                       "l2": f"inputs ({n * d * elem / 1e6:.0f} MB/rank) larger than the 126 MB L2; no explicit flush",
                       "parallelism": f"shard-parallel x{world} (LPT on m^2), library NCCL bcast + send/recv"},
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches,
            "clocks": clocks, "recall_at_10": recall,
            "parity_at_scale": parity,
            "stage_ms_untimed_step": stage_ms,
        }
        emit(line)
    if world > 1:
        dist.barrier()
        api.scalegann_comm_destroy(comm)
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
