#!/usr/bin/env python
"""First measurements toward SURVEY §8(f) NEXT-1 and NEXT-2 (GPU only, not part of bench.py).

NEXT-1 — search throughput: queries/s of `scalegann_search_eval` (batched greedy beam search,
a9 / K11) against recall@10, for beam widths 16..256, on the C1 graph (1M x 128, k = 4,
omega = 2, eps = 1.2, L = 128, R = 64).  Ground truth (K10) is computed once and passed in, so
the timed call is the beam search plus the recall count; CUDA events on the launching stream,
warm-up call first.

NEXT-1 also reports the distance-count proxy of search work (distances computed per
query, from the library's counter) and batch latency percentiles (CUDA events around each call;
batches of 1, 32 and 1024 queries).

NEXT-2 — selectivity sweep (Table 4 / Fig. 3): eps in {1.0, 1.005, 1.01, 1.02, 1.05,
1.1, 1.2, 1.5, 3.0} with omega = 2 (the squared-distance ratios d'/d of this 128-d data sit just
above 1, so eps binds below ~1.1 and the replica budget above), plus the split-only build
(omega = 1, no replicas): replication proportion
(replicas / n), device build time per step, recall@10 at beam 64.  The split-only graph is
searched both from the single global entry point and per shard with result merge
(`scalegann_search_eval_shards`, one beam of 64 per shard entry), as the paper's split-only
systems (GGNN / Extended CAGRA) search.

    python tools/sweep_next.py [--n 1000000] > gpurun_out/sweep_next.json
"""
from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2605_10135_b200 import api, datagen  # noqa: E402
from paper_2605_10135_b200.pipeline import BuildConfig, build_index  # noqa: E402


def timed_build(x, cfg, steps=2):
    build_index(x, cfg)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        idx = build_index(x, cfg)
    e1.record()
    torch.cuda.synchronize()
    return idx, e0.elapsed_time(e1) / steps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1_000_000)
    ap.add_argument("--nq", type=int, default=10_000)
    a = ap.parse_args()
    assert torch.cuda.is_available(), "GPU required"
    n = a.n
    x = datagen.sift_like(n, 128, device="cuda")
    q = datagen.sift_like(a.nq, 128, seed=datagen.DATA_SEED + datagen.QUERY_SEED_OFFSET, device="cuda")
    out = {"workload": f"C1 SIFT-shaped {n}x128 f32, k=4, L=128, R=64, {a.nq} queries", "next1_search": [],
           "next2_selectivity": []}

    # NEXT-2 sweep (also yields the eps = 1.2 graph for NEXT-1)
    gt = None
    base = None
    for omega, eps in [(2, 1.0), (2, 1.005), (2, 1.01), (2, 1.02), (2, 1.05), (2, 1.1), (2, 1.2), (2, 1.5), (2, 3.0),
                       (1, 1.0)]:
        cfg = BuildConfig(k=4, omega=omega, epsilon=eps, L=128, R=64)
        idx, ms = timed_build(x, cfg)
        if gt is None:
            _, gt, _ = api.scalegann_search_eval(x, idx.merged, idx.entry, q, topk=10, beam=64)
        _, _, rec, nd = api.scalegann_search_eval(x, idx.merged, idx.entry, q, topk=10, beam=64, gt=gt,
                                                  return_ndist=True)
        repl = sum(idx.counts["repl"])
        _, entries = api.scalegann_entry_points(idx.home, idx.primary_d, idx.sizes)
        _, _, rec_sh = api.scalegann_search_eval_shards(x, idx.merged, entries, q, topk=10, beam=64, gt=gt)
        out["next2_selectivity"].append({"omega": omega, "epsilon": eps, "replicas": repl,
                                         "replication_proportion": repl / n, "shard_sizes": idx.sizes,
                                         "build_ms": ms, "build_vectors_per_s": n / (ms / 1000.0),
                                         "recall_at_10_beam64": rec, "distances_per_query_beam64": nd / a.nq,
                                         "recall_at_10_beam64_per_shard_search": rec_sh})
        if omega == 2 and eps == 1.2:
            base = idx
        if omega == 1:   # split-only: per-shard search throughput vs recall (QPS-matched comparison)
            out["next2_split_only_search"] = []
            for beam in (16, 32, 64):
                api.scalegann_search_eval_shards(x, idx.merged, entries, q, topk=10, beam=beam, gt=gt)
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                for _ in range(3):
                    _, _, r = api.scalegann_search_eval_shards(x, idx.merged, entries, q, topk=10, beam=beam, gt=gt)
                e1.record()
                torch.cuda.synchronize()
                ms = e0.elapsed_time(e1) / 3
                out["next2_split_only_search"].append({"beam_per_shard": beam, "recall_at_10": r,
                                                       "ms_per_batch": ms, "qps": a.nq / (ms / 1000.0)})
        del idx
        torch.cuda.empty_cache()

    # NEXT-1 search throughput, distance counts and batch latency on the paper's default configuration
    for beam in (16, 32, 64, 128, 256):
        api.scalegann_search_eval(x, base.merged, base.entry, q, topk=10, beam=beam, gt=gt)   # warm-up
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 3
        e0.record()
        for _ in range(reps):
            _, _, rec, nd = api.scalegann_search_eval(x, base.merged, base.entry, q, topk=10, beam=beam, gt=gt,
                                                      return_ndist=True)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        lat = {}
        for bs, nb in ((1, 200), (32, 100), (1024, 10)):
            times = []
            for b in range(nb):
                qb = q[(b * bs) % (a.nq - bs):][:bs]
                gb = gt[(b * bs) % (a.nq - bs):][:bs]
                t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                t0.record()
                api.scalegann_search_eval(x, base.merged, base.entry, qb, topk=10, beam=beam, gt=gb)
                t1.record()
                torch.cuda.synchronize()
                times.append(t0.elapsed_time(t1))
            times.sort()
            lat[f"batch{bs}"] = {"p50_ms": times[len(times) // 2], "p99_ms": times[min(len(times) - 1,
                                                                                      int(0.99 * len(times)))]}
        out["next1_search"].append({"beam": beam, "recall_at_10": rec, "ms_per_batch": ms,
                                    "qps": a.nq / (ms / 1000.0), "distances_per_query": nd / a.nq,
                                    "latency": lat})
    print(json.dumps(out))


if __name__ == "__main__":
    main()
