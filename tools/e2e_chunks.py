"""Wall time of sparse_conv_forward_host (C2, N=128, s=0.95, pinned) for SC_HOST_CHUNKS=argv[1]."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1704_07724_b200 import datagen, sparseconv as sc  # noqa: E402

shp = datagen.C2
w, b = datagen.weights(shp)
dev = torch.device("cuda", 0)
conv = sc.SparseConv(torch.from_numpy(w).to(dev), torch.from_numpy(b).to(dev), shp.n, shp.c, shp.h, shp.w, 1, 1, 1)
h_in = torch.from_numpy(datagen.activations(shp, 0.95)).pin_memory()
h_out = torch.empty((shp.n, shp.k, shp.ho, shp.wo)).pin_memory()
for _ in range(3):
    conv.forward_host(h_in, h_out)
ts = []
for _ in range(5):
    t0 = time.perf_counter()
    for _ in range(10):
        conv.forward_host(h_in, h_out)
    ts.append((time.perf_counter() - t0) / 10 * 1e3)
print(os.environ.get("SC_HOST_CHUNKS"), "ms", [round(t, 3) for t in ts])
