"""Time and check every stage-2 variant that matches a config:
python tools/variant_sweep.py C2 0.95 "10 11 12 13 7 1" """
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
from paper_1704_07724_b200 import datagen, sparseconv as sc  # noqa: E402
from tools.probe_run import dev_time_us  # noqa: E402

cfg = sys.argv[1]
sps = [x if x == "channel" else float(x) for x in sys.argv[2].split(",")]
vids = [int(v) for v in sys.argv[3].split()]
shp = datagen.CONFIGS[cfg]
w, b = datagen.weights(shp)
for s in sps:
    xh = datagen.activations(shp, s)
    x = torch.from_numpy(xh).cuda()
    ref = {}
    for i in (0, shp.n - 1):
        ref[i] = oracle.conv_fp64(xh[i:i + 1], w, b, shp.stride, shp.pad, shp.groups)
    for v in vids:
        os.environ["SC_FORCE_VARIANT"] = str(v)
        conv = sc.SparseConv(torch.from_numpy(w).cuda(), torch.from_numpy(b).cuda(), shp.n, shp.c, shp.h, shp.w,
                             shp.stride, shp.pad, shp.groups)
        out = conv.forward(x)
        torch.cuda.synchronize()
        worst = 0.0
        for i, (r, mass) in ref.items():
            err = np.abs(out[i:i + 1].cpu().numpy().astype(np.float64) - r) / oracle.tolerance_sparse(mass)
            worst = max(worst, float(err.max()))
        t_c = dev_time_us(lambda: conv.compact(x))
        t_g = dev_time_us(lambda: conv.gather(shp.n, out))
        print(f"{cfg} s={s} variant={conv.variant} err/tol={worst:.3g} compact={t_c:.1f}us gather={t_g:.1f}us",
              flush=True)
        del conv
