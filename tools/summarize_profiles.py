"""Summarise a round's ncu captures into profiles/ (tracked):
  python tools/summarize_profiles.py TAG M
reads gpurun_out/TAG_launches.csv (launch list of bench.py --profile-steps), gpurun_out/TAG_knn_full.ncu-rep
(ncu --set full of the main distance-kernel launch at shard size M), gpurun_out/prune_full.ncu-rep, and
gpurun_out/TAG_bench.json / TAG_ref.json; writes profiles/TAG_*.txt|json and profiles/knn_dram_bytes.json."""
import collections
import csv
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G = os.path.join(ROOT, "gpurun_out")
P = os.path.join(ROOT, "profiles")


def raw(rep, kernel_regex=None):
    cmd = ["ncu", "-i", rep, "--page", "raw", "--csv"]
    if kernel_regex:
        cmd += ["-k", kernel_regex]
    out = subprocess.run(cmd, capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    return [{h: (v, u) for h, v, u in zip(hdr, r, units)} for r in rows[2:]]


def num(d, k):
    return float(d[k][0].replace(",", ""))


def main():
    tag, m = sys.argv[1], int(sys.argv[2])
    os.makedirs(P, exist_ok=True)
    # launch list
    rows = [r for r in csv.reader(open(os.path.join(G, f"{tag}_launches.csv"))) if len(r) > 5]
    hdr = rows[0]
    ix = {h: i for i, h in enumerate(hdr)}
    data = [r for r in rows[1:] if r[ix["Metric Name"]] == "gpu__time_duration.sum"]
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in data:
        k = r[ix["Kernel Name"]].split("(")[0].replace("void ", "")
        agg[k][0] += 1
        agg[k][1] += float(r[ix["Metric Value"]].replace(",", ""))
    tot = sum(v[1] for v in agg.values())
    lines = [f"# ncu launch list of `python bench.py --profile-steps --steps 1 --warmup 3` ({tag}, one B200)",
             f"# --metrics gpu__time_duration.sum --clock-control none; {len(data)} launches (3 warm-up + 1 step);",
             "# cold-cache serialised times: compare SHARES with the bench's live numbers, not absolutes", "",
             f"{'kernel':60s} {'launches':>8s} {'total ns':>14s} {'share':>7s}"]
    for k, (n, v) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        lines.append(f"{k[:60]:60s} {n:8d} {v:14.0f} {100 * v / tot:6.1f}%")
    open(os.path.join(P, f"{tag}_bench_launches.txt"), "w").write("\n".join(lines) + "\n")
    # distance kernel
    d = raw(os.path.join(G, f"{tag}_knn_full.ncu-rep"))[0]
    flops = 2.0 * m * m * 128
    keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
            "sm__ops_path_tensor_op_utchmma_src_fp16_dst_fp32_sparsity_off.avg.pct_of_peak_sustained_elapsed",
            "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__inst_executed.avg.per_cycle_elapsed",
            "smsp__inst_executed.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
            "sm__cycles_elapsed.avg.per_second", "launch__registers_per_thread", "launch__grid_size",
            "launch__block_size", "smsp__mem_tensor_reads_op_ldt.sum.pct_of_peak_sustained_elapsed",
            "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"]
    dur = num(d, "gpu__time_duration.sum")
    out = [f"# ncu --set full --clock-control none of the main distance-kernel launch ({tag})",
           f"# python tools/profile_knn.py --m {m} --reps 1 (-k regex:knn_tc -s 0 -c 1): the bench's largest shard",
           f"# kernel: {d['Kernel Name'][0]}",
           f"# algorithmic 2 m^2 d = {flops:.4e} flop -> {flops / (dur / 1e3) / 1e12:.1f} TFLOP/s under ncu", ""]
    out += [f"{k:88s} {d[k][0]:>22s} {d[k][1]}" for k in keys if k in d]
    open(os.path.join(P, f"{tag}_knn_ncu_full.txt"), "w").write("\n".join(out) + "\n")
    rd, wr = num(d, "dram__bytes_read.sum"), num(d, "dram__bytes_write.sum")
    scale = 1e9 if d["dram__bytes_read.sum"][1].startswith("G") else 1e6
    tp = d.get("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", ("nan", ""))[0]
    json.dump({"kernel": d["Kernel Name"][0], "m": m, "dram_bytes_per_launch": (rd + wr) * scale,
               "tensor_pipe_active_pct": float(tp.replace(",", "")),
               "dram_read_bytes": rd * scale, "dram_write_bytes": wr * scale,
               "source": f"profiles/{tag}_knn_ncu_full.txt (ncu --set full)",
               "note": "writes are per-row candidate appends evicted from L2; operand reads stay mostly in L2"},
              open(os.path.join(P, "knn_dram_bytes.json"), "w"), indent=1)
    # prune / reverse
    pr = os.path.join(G, "prune_full.ncu-rep")
    if os.path.exists(pr):
        out = [f"# ncu --set full of a6 prune + a7 reverse on one 450000-row shard (L=128, R=64) ({tag})",
               "# algorithmic bytes per node (SURVEY 8(d)): prune 4(L + L^2 + R) + 4L + 4R = 67 328 B;"
               " reverse ~ 30 R = 1 920 B", ""]
        for kd in raw(pr):
            name = kd["Kernel Name"][0].split("(")[0]
            t = num(kd, "gpu__time_duration.sum")
            unit = kd["gpu__time_duration.sum"][1]
            ms = t / 1e3 if unit == "us" else t
            per_node = 67328 if "prune" in name else 1920
            alg = 450000 * per_node / (ms / 1e3) / 1e9
            out.append(f"{name}: {ms:.3f} ms, algorithmic {alg:.0f} GB/s "
                       f"({100 * alg / 6550.4:.1f}% of 6550.4 GB/s measured HBM)")
            for k in ["dram__bytes_read.sum", "dram__bytes_write.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
                      "lts__t_bytes.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
                      "sm__inst_executed.avg.per_cycle_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
                      "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"]:
                if k in kd:
                    out.append(f"    {k:80s} {kd[k][0]:>18s} {kd[k][1]}")
        open(os.path.join(P, f"{tag}_prune_reverse_ncu.txt"), "w").write("\n".join(out) + "\n")
    for f in (f"{tag}_bench.json", f"{tag}_ref.json"):
        if os.path.exists(os.path.join(G, f)):
            shutil.copy(os.path.join(G, f), os.path.join(P, f))
    print("\n".join(lines[:12]))


if __name__ == "__main__":
    main()
