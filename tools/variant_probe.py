"""Run one forced stage-2 variant on a tiny case of a config and compare with
the oracle.  Usage: SC_FORCE_VARIANT=v python tools/variant_probe.py C2 0.95 n"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
from paper_1704_07724_b200 import datagen, sparseconv as sc  # noqa: E402

cfg, s, n = sys.argv[1], float(sys.argv[2]), int(sys.argv[3])
shp = datagen.CONFIGS[cfg].with_batch(n)
x = datagen.activations(shp, s if cfg != "C3" else "channel")
w, b = datagen.weights(shp)
conv = sc.SparseConv(torch.from_numpy(w).cuda(), torch.from_numpy(b).cuda(), n, shp.c, shp.h, shp.w, shp.stride,
                     shp.pad, shp.groups)
print("variant", conv.variant, flush=True)
out = conv.forward(torch.from_numpy(x).cuda())
torch.cuda.synchronize()
ref, mass = oracle.conv_fp64(x, w, b, shp.stride, shp.pad, shp.groups)
r = np.abs(out.cpu().numpy() - ref) / oracle.tolerance_sparse(mass)
print(cfg, s, n, "max err/tol", r.max(), "ok" if r.max() <= 1 else "FAIL", flush=True)
