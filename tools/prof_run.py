"""Small driver for ncu captures: runs sparse_conv_forward (and the dense
path if present) a few times on one config.  Usage:
  python tools/prof_run.py [C2] [0.95] [reps]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1704_07724_b200 import datagen, sparseconv as sc  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
s = float(sys.argv[2]) if len(sys.argv) > 2 else 0.95
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
dense = len(sys.argv) > 4 and sys.argv[4] == "dense"
shp = datagen.CONFIGS[cfg]
x = torch.from_numpy(datagen.activations(shp, s)).cuda()
w, b = datagen.weights(shp)
conv = sc.SparseConv(torch.from_numpy(w).cuda(), torch.from_numpy(b).cuda(), shp.n, shp.c, shp.h, shp.w,
                     shp.stride, shp.pad, shp.groups)
out = torch.empty((shp.n,) + conv.out_shape, device="cuda")
for _ in range(reps):
    conv.forward(x, out)
    if dense:
        conv.dense_forward(x, out)
torch.cuda.synchronize()
print("ok", conv.variant)
