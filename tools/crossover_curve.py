"""Sparse forward vs tcgen05 dense forward vs forward_auto over a sparsity sweep
(graph-timed, L2-warm), with the calibrated s*: the crossover curve of SURVEY 8f row f3.
python tools/crossover_curve.py C2 C4a C4b"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1704_07724_b200 import datagen, sparseconv as sc  # noqa: E402
from tools.probe_run import dev_time_us  # noqa: E402

SWEEP = [0.5, 0.7, 0.8, 0.9, 0.93, 0.95, 0.97, 0.98, 0.99, 0.995]
for cfg in sys.argv[1:] or ["C2"]:
    shp = datagen.CONFIGS[cfg]
    w, b = datagen.weights(shp)
    conv = sc.SparseConv(torch.from_numpy(w).cuda(), torch.from_numpy(b).cuda(), shp.n, shp.c, shp.h, shp.w,
                         shp.stride, shp.pad, shp.groups)
    out = torch.empty((shp.n, shp.k, shp.ho, shp.wo), device="cuda")
    s_star = conv.calibrate_crossover(shp.n)
    print(f"{cfg} variant={conv.variant[1]} calibrated s*={s_star:.4f}")
    print(f"{'s':>6} {'sparse_us':>10} {'dense_us':>9} {'auto_us':>8} auto_path")
    for s in SWEEP:
        x = torch.from_numpy(datagen.activations(shp, s)).cuda()
        ts = dev_time_us(lambda: conv.forward(x, out), reps=5)
        td = dev_time_us(lambda: conv.dense_forward(x, out), reps=5)
        ta = dev_time_us(lambda: conv.forward_auto(x, out), reps=5)
        path = "sparse" if conv.last_path()[0] == sc.SC_PATH_SPARSE else "dense"
        print(f"{s:6.3f} {ts:10.1f} {td:9.1f} {ta:8.1f} {path}", flush=True)
