"""Per-stage device times (compaction, gather, forward) of the paper Table 2 layers at N=128."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1704_07724_b200 import datagen, sparseconv as sc  # noqa: E402
from tools.probe_run import dev_time_us  # noqa: E402

for shp, s in datagen.table2_shapes(n=128):
    x = torch.from_numpy(datagen.activations(shp, s)).cuda()
    w, b = datagen.weights(shp)
    conv = sc.SparseConv(torch.from_numpy(w).cuda(), torch.from_numpy(b).cuda(), shp.n, shp.c, shp.h, shp.w,
                         shp.stride, shp.pad, shp.groups)
    out = conv.forward(x)
    tc = dev_time_us(lambda: conv.compact(x))
    tg = dev_time_us(lambda: conv.gather(shp.n, out))
    tf = dev_time_us(lambda: conv.forward(x, out))
    print(f"{shp.name:24s} compact {tc:7.1f} gather {tg:7.1f} forward {tf:7.1f}", flush=True)
