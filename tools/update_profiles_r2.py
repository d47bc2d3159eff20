"""Refresh profiles/ from gpurun_out/m/ (tools/gpu_r2_measure.sh): launch list, ncu
summaries of the gather and the dense GEMM, the gather's traffic figures for bench.py's
roofline object, the FFMA/FFMA2 census and the bench lines."""
import csv
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from update_profiles import KEEP, raw, to_bytes  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G = os.path.join(ROOT, "gpurun_out", "m")
P = os.path.join(ROOT, "profiles")
EXTRA = ["l1tex__m_xbar2l1tex_read_bytes.sum", "lts__t_sectors_srcunit_tex_op_write.sum",
         "lts__t_sectors_srcunit_tex_op_read.sum", "sm__mem_tensor_cycles_active", "gpc__cycles_elapsed.max",
         "lts__t_sectors_srcunit_tex.avg.per_cycle_elapsed", "sm__inst_executed_pipe_tc"]


def summary(rep, title, path):
    rows = raw(rep)
    h, u = rows[0], rows[1]
    vals = {}
    with open(path, "w") as f:
        f.write(title)
        for v in rows[2:]:
            f.write(f"\n## launch: {v[h.index('Kernel Name')][:100]}\n")
            for i, name in enumerate(h):
                if any(name.startswith(k) for k in KEEP + EXTRA) and not name.endswith("_not_issued"):
                    f.write(f"{name} [{u[i]}] = {v[i]}\n")
                    vals[name] = (u[i], v[i])
    return vals


def num(vals, key):
    u, v = vals[key]
    try:
        return to_bytes(u, v)
    except KeyError:
        return float(v.replace(",", ""))


def main():
    tag = "r2"
    rows = [r for r in csv.reader(open(os.path.join(G, "launches.csv"))) if len(r) > 10]
    h = rows[0]
    ki, mi, vi, ii = h.index('Kernel Name'), h.index('Metric Name'), h.index('Metric Value'), h.index('ID')
    d = {}
    for r in rows[1:]:
        d.setdefault((int(r[ii]), r[ki].split('(')[0]), {})[r[mi]] = r[vi]
    with open(os.path.join(P, f"{tag}_launches_bench_C2_s095.csv"), "w") as f:
        f.write("# ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum "
                "--clock-control none (cold cache, serialised) of: python bench.py --steps 2 --warmup 3 --no-sweep "
                "--no-cpu-baseline\n")
        f.write("id,kernel,duration_ns,dram_read_bytes,dram_write_bytes,lts_bytes\n")
        for (i, k), m in sorted(d.items()):
            f.write(f"{i},{k},{m.get('gpu__time_duration.sum')},{m.get('dram__bytes_read.sum')},"
                    f"{m.get('dram__bytes_write.sum')},{m.get('lts__t_bytes.sum')}\n")
    g = summary(os.path.join(G, "gather_C2.ncu-rep"),
                f"# ncu --set full --clock-control none: stage-2 gather kernel (V21), C2 (N=128) s=0.95, B200 ({tag})\n",
                os.path.join(P, f"{tag}_gather_C2_s095_raw_summary.txt"))
    summary(os.path.join(G, "dense_C2.ncu-rep"),
            f"# ncu --set full --clock-control none: dense tcgen05 TF32 GEMM (persistent), C2 N=128, B200 ({tag})\n",
            os.path.join(P, f"{tag}_dense_C2_raw_summary.txt"))
    bench = json.loads(open(os.path.join(G, "bench_C2.log")).read().strip().splitlines()[-1])
    variant = bench["config"]["variant"]
    dram = num(g, "dram__bytes_read.sum") + num(g, "dram__bytes_write.sum")
    l2w = num(g, "lts__t_sectors_srcunit_tex_op_write.sum") * 32
    l2sm = num(g, "l1tex__m_xbar2l1tex_read_bytes.sum")
    json.dump({variant: {"traffic_bytes": int(num(g, "dram__bytes_read.sum") + l2w), "dram_bytes": int(dram),
                         "l2_write_bytes": int(l2w), "l2_to_sm_bytes": int(l2sm)},
               "_note": "one gather launch (C2 N=128 s=0.95) from ncu --set full --clock-control none: traffic_bytes = "
                        "dram__bytes_read.sum + 32 x lts__t_sectors_srcunit_tex_op_write.sum (the outputs are still "
                        "L2-resident when the launch ends, so DRAM writes undercount them); l2_to_sm_bytes = "
                        "l1tex__m_xbar2l1tex_read_bytes.sum (weight slices streamed by TMA into every CTA's ring, "
                        "plus the stage-1 streams)"},
              open(os.path.join(P, "gather_traffic.json"), "w"), indent=1)
    print("variant", variant, "dram", dram, "l2 writes", l2w, "l2->sm", l2sm)


if __name__ == "__main__":
    main()
