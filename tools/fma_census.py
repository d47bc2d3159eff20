"""Hardware count of the FMAs the stage-2 kernel executes (the north star's
"fraction of MACs skipped"): one sparse forward per workload, run
under ncu with the FFMA / FFMA2 thread-instruction counters on the gather
launches; this driver writes the exact and dense MAC counts of the same inputs.

  ncu --metrics smsp__sass_thread_inst_executed_op_ffma_pred_on.sum,\
smsp__sass_thread_inst_executed_op_ffma2_pred_on.sum,gpu__time_duration.sum \
      -k regex:gather_fast --csv --log-file gpurun_out/fma_census.csv \
      python tools/fma_census.py gpurun_out/fma_census_counts.jsonl
  python tools/fma_census.py --summarize gpurun_out/fma_census_counts.jsonl gpurun_out/fma_census.csv out.json
"""
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

WORKLOADS = [("C1", 0.9), ("C2", 0.9), ("C2", 0.95), ("C2", 0.99), ("C3", "channel"), ("C4a", 0.9),
             ("C4a", 0.95), ("C4a", 0.99), ("C4b", 0.9), ("C4b", 0.95), ("C4b", 0.99)]


def run(path):
    import torch
    import bench
    from paper_1704_07724_b200 import datagen, sparseconv as sc
    with open(path, "w") as f:
        for cfg, s in WORKLOADS:
            shp = datagen.CONFIGS[cfg]
            x = torch.from_numpy(datagen.activations(shp, s)).cuda()
            w, b = datagen.weights(shp)
            conv = sc.SparseConv(torch.from_numpy(w).cuda(), torch.from_numpy(b).cuda(), shp.n, shp.c, shp.h,
                                 shp.w, shp.stride, shp.pad, shp.groups)
            conv.forward(x)
            torch.cuda.synchronize()
            dense, exact, nnz = bench.mac_counts(x, shp)
            f.write(json.dumps({"workload": f"{cfg} s={s}", "variant": conv.variant[1], "dense_macs": dense,
                                "exact_nonzero_macs": exact, "nnz": nnz}) + "\n")
            del conv


def summarize(counts_path, csv_path, out_path):
    counts = [json.loads(l) for l in open(counts_path)]
    rows = [r for r in csv.reader(open(csv_path)) if len(r) > 5]
    h = rows[0]
    ik, im, iv = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
    iid = h.index("ID")
    per = {}
    for r in rows[1:]:
        if "gather_fast" not in r[ik]:
            continue
        per.setdefault(r[iid], {})[r[im]] = float(r[iv].replace(",", ""))
    launches = [per[k] for k in sorted(per, key=int)]
    assert len(launches) == len(counts), (len(launches), len(counts))
    out = []
    for c, m in zip(counts, launches):
        ffma = m["smsp__sass_thread_inst_executed_op_ffma_pred_on.sum"]
        ffma2 = m["smsp__sass_thread_inst_executed_op_ffma2_pred_on.sum"]
        executed = ffma + 2 * ffma2
        out.append(dict(c, ffma_thread_inst=int(ffma), ffma2_thread_inst=int(ffma2), executed_lane_fmas=int(executed),
                        wasted_fma_factor=round(executed / c["exact_nonzero_macs"], 4),
                        skipped_vs_dense_exact=round(1 - c["exact_nonzero_macs"] / c["dense_macs"], 5),
                        skipped_vs_dense_executed=round(1 - executed / c["dense_macs"], 5),
                        gather_us_ncu=round(m["gpu__time_duration.sum"] / 1e3, 2)))
    with open(out_path, "w") as f:
        json.dump({"source": "ncu --metrics smsp__sass_thread_inst_executed_op_ffma{,2}_pred_on.sum on the stage-2 "
                             "launches (one per workload, cold cache); executed lane-FMAs = FFMA + 2 x FFMA2",
                   "workloads": out}, f, indent=1)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    if sys.argv[1] == "--summarize":
        summarize(*sys.argv[2:5])
    else:
        run(sys.argv[1])
