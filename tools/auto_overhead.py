"""Overhead of sparse_conv_forward_auto over the path it picks (f3): graph-timed
auto vs forward / dense_forward on C2 (N=128), with the crossover forced each
way.  Run under ncu for the per-kernel split (gated-off kernels exit at once)."""
import json
import sys

import torch

sys.path.insert(0, ".")
from bench import graph_time_us  # noqa: E402
from paper_1704_07724_b200 import datagen, sparseconv as sc  # noqa: E402

dev = torch.device("cuda", 0)
shp = datagen.C2
w, b = datagen.weights(shp)
conv = sc.SparseConv(torch.from_numpy(w).to(dev), torch.from_numpy(b).to(dev), shp.n, shp.c, shp.h, shp.w, 1, 1, 1)
x = torch.from_numpy(datagen.activations(shp, 0.99)).to(dev)
out = torch.empty((shp.n, shp.k, shp.ho, shp.wo), device=dev)
st = torch.cuda.Stream(dev)
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
res = {}
res["sparse"] = graph_time_us(torch, st, lambda: conv.forward(x, out, stream=st), reps)
res["dense"] = graph_time_us(torch, st, lambda: conv.dense_forward(x, out, stream=st), reps)
conv.crossover = 0.0
res["auto_forced_sparse"] = graph_time_us(torch, st, lambda: conv.forward_auto(x, out, stream=st), reps)
conv.crossover = 1.0
res["auto_forced_dense"] = graph_time_us(torch, st, lambda: conv.forward_auto(x, out, stream=st), reps)
print(json.dumps({k: round(v, 2) for k, v in res.items()}))
