"""Run the C5 chain once fused and once unfused (for ncu launch lists)."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1704_07724_b200 import datagen, sparseconv as sc
n = int(sys.argv[1]) if len(sys.argv) > 1 else 128
layers = [shp.with_batch(n) for shp in datagen.C5_LAYERS]
weights = datagen.c5_weights()
convs = [sc.SparseConv(torch.from_numpy(w).cuda(), torch.from_numpy(b).cuda(), n, shp.c, shp.h, shp.w, shp.stride,
                       shp.pad, shp.groups, fuse_relu=li + 1 < len(layers)) for li, (shp, (w, b)) in enumerate(zip(layers, weights))]
x = torch.from_numpy(datagen.activations(layers[0], datagen.C5_FIRST_SPARSITY)).cuda()
outs = [torch.empty((n,) + c.out_shape, device="cuda") for c in convs]
for _ in range(2):
    sc.chain_forward(convs, x, [None, None, outs[-1]])
    for li, c in enumerate(convs):
        c.forward(x if li == 0 else outs[li - 1], outs[li])
torch.cuda.synchronize()
print("ok")
