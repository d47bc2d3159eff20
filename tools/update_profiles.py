"""Refresh profiles/ from a gpurun_out/ produced by tools/gpu_calls/gpu_final.sh:
launch list, gather/compaction ncu summaries, gather DRAM traffic, bench lines."""
import csv
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G = os.path.join(ROOT, "gpurun_out")
P = os.path.join(ROOT, "profiles")
tag = sys.argv[1] if len(sys.argv) > 1 else "r1"

KEEP = ['gpu__time_duration.sum', 'sm__pipe_tensor', 'sm__pipe_tc', 'lts__t_bytes.sum', 'lts__throughput.avg.pct', 'dram__bytes_read.sum', 'dram__bytes_write.sum', 'smsp__inst_executed.sum',
        'launch__registers_per_thread', 'launch__grid_size', 'launch__block_size',
        'sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active',
        'sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active',
        'l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum', 'l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum',
        'l1tex__data_pipe_lsu_wavefronts_mem_shared.sum', 'smsp__sass_thread_inst_executed_op_ffma_pred_on.sum',
        'sm__warps_active.avg.pct_of_peak_sustained_active', 'smsp__average_warps_issue_stalled',
        'smsp__issue_active.avg.pct_of_peak_sustained_active', 'sm__throughput.avg.pct_of_peak_sustained_elapsed']


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    return list(csv.reader(out.splitlines()))


def summary(rep, title, path):
    rows = raw(rep)
    h, u = rows[0], rows[1]
    with open(path, "w") as f:
        f.write(title)
        for v in rows[2:]:
            f.write(f"\n## launch: {v[h.index('Kernel Name')][:100]}\n")
            for i, name in enumerate(h):
                if any(name.startswith(k) for k in KEEP) and not name.endswith("_not_issued"):
                    f.write(f"{name} [{u[i]}] = {v[i]}\n")
    return rows


def to_bytes(unit, val):
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[unit]
    return float(val.replace(",", "")) * scale


def main():
    rows = [r for r in csv.reader(open(os.path.join(G, "launches.csv"))) if len(r) > 10]
    h = rows[0]
    ki, mi, vi, ii = h.index('Kernel Name'), h.index('Metric Name'), h.index('Metric Value'), h.index('ID')
    d = {}
    for r in rows[1:]:
        d.setdefault((int(r[ii]), r[ki].split('(')[0]), {})[r[mi]] = r[vi]
    with open(os.path.join(P, f"{tag}_launches_bench_C2_s095.csv"), "w") as f:
        f.write("# ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none "
                "(cold cache, serialised) of: python bench.py --steps 2 --warmup 3 --no-sweep --no-cpu-baseline\n")
        f.write("id,kernel,duration_ns,dram_read_bytes,dram_write_bytes\n")
        for (i, k), m in sorted(d.items()):
            f.write(f"{i},{k},{m.get('gpu__time_duration.sum')},{m.get('dram__bytes_read.sum')},"
                    f"{m.get('dram__bytes_write.sum')}\n")
    g = summary(os.path.join(G, "gather_full.ncu-rep"),
                f"# ncu --set full --clock-control none: stage-2 gather kernel, C2 (N=128) s=0.95, B200 ({tag})\n",
                os.path.join(P, f"{tag}_gather_C2_s095_raw_summary.txt"))
    summary(os.path.join(G, "compact_full.ncu-rep"),
            f"# ncu --set full --clock-control none: stage-1 compaction kernels, C2 s=0.95, B200 ({tag})\n",
            os.path.join(P, f"{tag}_compact_C2_s095_raw_summary.txt"))
    if os.path.exists(os.path.join(G, "dense_full.ncu-rep")):
        summary(os.path.join(G, "dense_full.ncu-rep"),
                f"# ncu --set full --clock-control none: dense tcgen05 TF32 GEMM (persistent), C2 N=128, B200 ({tag})\n",
                os.path.join(P, f"{tag}_dense_C2_raw_summary.txt"))
    for src, dst in (("crossover.txt", f"{tag}_crossover_C2_C4a_C4b.txt"), ("auto_overhead.txt", f"{tag}_auto_overhead_C2.txt"),
                     ("bench_bwd.log", f"{tag}_backward_C2.jsonl")):
        if os.path.exists(os.path.join(G, src)) and os.path.getsize(os.path.join(G, src)) > 0:
            shutil.copy(os.path.join(G, src), os.path.join(P, dst))
    h, u, v = g[0], g[1], g[2]
    traffic = to_bytes(u[h.index('dram__bytes_read.sum')], v[h.index('dram__bytes_read.sum')]) + \
        to_bytes(u[h.index('dram__bytes_write.sum')], v[h.index('dram__bytes_write.sum')])
    kname = v[h.index('Kernel Name')]
    bench = json.loads(open(os.path.join(G, "bench.log")).read().strip().splitlines()[-1])
    variant = bench["config"]["variant"]
    json.dump({variant: int(traffic),
               "_note": f"dram__bytes_read.sum + dram__bytes_write.sum of one gather launch ({kname[:60]}, C2 N=128 "
                        "s=0.95) from ncu --set full --clock-control none; ncu flushes caches before the launch and "
                        "the 33 MB of outputs are still L2-resident when it ends"},
              open(os.path.join(P, "gather_traffic.json"), "w"), indent=1)
    for src, dst in (("bench.log", f"{tag}_bench_C2.jsonl"), ("bench_c5.log", f"{tag}_bench_C5.jsonl"),
                     ("bench_ref.log", f"{tag}_bench_reference.jsonl")):
        shutil.copy(os.path.join(G, src), os.path.join(P, dst))
    print("traffic", traffic, "variant", variant)


if __name__ == "__main__":
    main()
