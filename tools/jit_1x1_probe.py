"""1x1 shapes without a shipped variant: the run-time generated default tiling (csrc/jit.cu
choose(): KL = 6 / 8 one-row tiles for Kg >= 150) against the round-1 rule (KL = 4, the
tallest tile in 140 registers, forced through SC_JIT_FORCE), whole forward, graph-timed;
image 0 checked against the oracle for both.
Usage: python tools/jit_1x1_probe.py [s] ["C,H,K;C,H,K" shapes] ["TY,KL,...;TY,KL,..." extra forced sets]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
from paper_1704_07724_b200 import datagen, sparseconv as sc  # noqa: E402
from tools.probe_run import dev_time_us  # noqa: E402

s = float(sys.argv[1]) if len(sys.argv) > 1 else 0.9
dev = torch.device("cuda", 0)
# (C, H = W, K): Inception-style 1x1 layers on 7-17 wide planes
SHAPES = [(512, 14, 160), (512, 14, 256), (528, 14, 256), (480, 14, 208), (832, 7, 384), (1024, 7, 512),
          (768, 17, 192), (768, 17, 160), (256, 12, 150), (512, 10, 300)]
if len(sys.argv) > 2 and sys.argv[2]:
    SHAPES = [tuple(int(v) for v in t.split(",")) for t in sys.argv[2].split(";")]
EXTRA = sys.argv[3].split(";") if len(sys.argv) > 3 else []


def old_rule(ho, wo):
    ty = min((140 - 4) // (4 * wo), ho)
    tiles = (ho + ty - 1) // ty
    return (ho + tiles - 1) // tiles


for c, hw, k in SHAPES:
    shp = datagen.ConvShape(f"1x1_{c}_{hw}_{k}", 7000 + k + hw, 128, c, hw, hw, k, 1, 1, 1, 0, 1)
    w, b = datagen.weights(shp)
    xh = datagen.activations(shp, s)
    x = torch.from_numpy(xh).to(dev)
    out = torch.empty((shp.n, shp.k, shp.ho, shp.wo), device=dev)
    ref, mass = oracle.conv_fp64(xh[:1], w, b, 1, 0, 1)
    row = [f"C={c} W={hw} K={k}"]
    for force in [None, f"{old_rule(shp.ho, shp.wo)},4,11,1,16,2,3,254"] + EXTRA:
        if force:
            os.environ["SC_JIT_FORCE"] = force
        else:
            os.environ.pop("SC_JIT_FORCE", None)
        try:
            conv = sc.SparseConv(torch.from_numpy(w).to(dev), torch.from_numpy(b).to(dev), shp.n, shp.c, shp.h, shp.w)
        except sc.SparseConvError as e:
            row.append(f"{force}: rejected ({e})")
            continue
        conv.forward(x, out)
        torch.cuda.synchronize()
        err = float((np.abs(out[:1].cpu().numpy() - ref) / oracle.tolerance_sparse(mass)).max())
        t = dev_time_us(lambda: conv.forward(x, out), reps=10)
        row.append(f"{force or 'default'} {conv.variant[1]} {t:.1f}us err/tol {err:.3f}")
        del conv
    print(" | ".join(row), flush=True)
os.environ.pop("SC_JIT_FORCE", None)
