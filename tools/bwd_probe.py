"""One sparse_conv_backward on C2 (N=128) for ncu captures of the backward kernels."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1704_07724_b200 import datagen, sparseconv as sc  # noqa: E402

s = float(sys.argv[1]) if len(sys.argv) > 1 else 0.95
dev = torch.device("cuda", 0)
shp = datagen.C2
w, b = datagen.weights(shp)
conv = sc.SparseConv(torch.from_numpy(w).to(dev), torch.from_numpy(b).to(dev), shp.n, shp.c, shp.h, shp.w, 1, 1, 1)
x = torch.from_numpy(datagen.activations(shp, s)).to(dev)
d = torch.from_numpy(np.random.default_rng(1).standard_normal((shp.n, shp.k, shp.ho, shp.wo)).astype(np.float32)).to(dev)
for _ in range(2):
    conv.backward(x, d)
torch.cuda.synchronize()
print("ok")
