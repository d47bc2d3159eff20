"""One dense_conv_forward on C2 (N=128) for ncu captures."""
import sys

import torch

sys.path.insert(0, ".")
from paper_1704_07724_b200 import datagen, sparseconv as sc  # noqa: E402

dev = torch.device("cuda", 0)
shp = datagen.C2
w, b = datagen.weights(shp)
conv = sc.SparseConv(torch.from_numpy(w).to(dev), torch.from_numpy(b).to(dev), shp.n, shp.c, shp.h, shp.w, 1, 1, 1)
x = torch.from_numpy(datagen.activations(shp, 0.95)).to(dev)
for _ in range(2):
    conv.dense_forward(x)
torch.cuda.synchronize()
print("ok")
