"""Stage-2 kernel choice, plan creation time and graph-timed forward (run-time generated
variant vs the generic kernel vs the dense path) for shapes without shipped variants.
Usage: python tools/jit_probe.py [s]"""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1704_07724_b200 import datagen, sparseconv as sc  # noqa: E402
from tools.probe_run import dev_time_us  # noqa: E402

s = float(sys.argv[1]) if len(sys.argv) > 1 else 0.95
dev = torch.device("cuda", 0)
print("jit available", sc.lib().sc_jit_available())
SHAPES = [("resnet conv2_x 3x3", (128, 64, 56, 56, 64, 3, 3, 1, 1, 1)),
          ("vgg conv4 3x3 W=20", (128, 256, 20, 20, 256, 3, 3, 1, 1, 1)),
          ("stride-2 3x3 W=32", (128, 64, 32, 32, 128, 3, 3, 2, 1, 1)),
          ("1x1 W=17", (128, 256, 17, 17, 128, 1, 1, 1, 0, 1))]
for label, a in SHAPES:
    shp = datagen.ConvShape("x", 999, *a)
    w, b = datagen.weights(shp)
    x = torch.from_numpy(datagen.activations(shp, s)).to(dev)
    out = torch.empty((shp.n, shp.k, shp.ho, shp.wo), device=dev)
    row = [label]
    for env in (None, "1"):
        if env:
            os.environ["SC_NO_JIT"] = env
        else:
            os.environ.pop("SC_NO_JIT", None)
        t0 = time.time()
        conv = sc.SparseConv(torch.from_numpy(w).to(dev), torch.from_numpy(b).to(dev), shp.n, shp.c, shp.h, shp.w,
                             shp.stride, shp.pad, shp.groups)
        tc = time.time() - t0
        t = dev_time_us(lambda: conv.forward(x, out), reps=3)
        row.append(f"{conv.variant[1]}: create {tc:.2f}s fwd {t:.1f}us")
        if env:
            row.append(f"dense {dev_time_us(lambda: conv.dense_forward(x, out), reps=3):.1f}us")
    print(" | ".join(row), flush=True)
os.environ.pop("SC_NO_JIT", None)
