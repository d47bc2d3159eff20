"""Run stage 1 (sparse_conv_compact) of one config a few times (for ncu captures of the
count / emit kernels).  Usage: python tools/stage1_probe.py [cfg] [s] [reps]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1704_07724_b200 import datagen, sparseconv as sc  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
s = float(sys.argv[2]) if len(sys.argv) > 2 else 0.95
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
shp = datagen.CONFIGS[cfg]
w, b = datagen.weights(shp)
x = torch.from_numpy(datagen.activations(shp, s)).cuda()
conv = sc.SparseConv(torch.from_numpy(w).cuda(), torch.from_numpy(b).cuda(), shp.n, shp.c, shp.h, shp.w, shp.stride,
                     shp.pad, shp.groups)
for _ in range(reps):
    conv.compact(x)
torch.cuda.synchronize()
print("ok", conv.variant)
