"""Quick GPU probe: FMA-pipe rates and per-stage timings of the sparse path on
C2 (AlexNet conv3, N=128).  Prints plain text; not a bench line."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1704_07724_b200 import datagen, sparseconv as sc  # noqa: E402


def timeit(fn, reps=20, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    ts.sort()
    return ts[len(ts) // 2]


def main():
    for kind, name in ((0, "FFMA"), (1, "FFMA2"), (2, "FFMA2+int")):
        print(f"probe {name}: {sc.probe_fma(kind):.1f} lane-FMA/clk/SM")
    for cfg in ("C2", "C4a", "C3", "C1", "C4b"):
        for s in (0.9, 0.95, 0.99) if cfg != "C3" else ("channel",):
            shp = datagen.CONFIGS[cfg]
            x = torch.from_numpy(datagen.activations(shp, s)).cuda()
            w, b = datagen.weights(shp)
            conv = sc.SparseConv(torch.from_numpy(w).cuda(), torch.from_numpy(b).cuda(), shp.n, shp.c, shp.h,
                                 shp.w, shp.stride, shp.pad, shp.groups)
            out = conv.forward(x)
            t_c = timeit(lambda: conv.compact(x))
            t_g = timeit(lambda: conv.gather(shp.n, out))
            t_f = timeit(lambda: conv.forward(x, out))
            print(f"{cfg} s={s} variant={conv.variant} compact={t_c:.1f}us gather={t_g:.1f}us forward={t_f:.1f}us")
            if cfg in ("C1", "C4b"):
                break


if __name__ == "__main__":
    main()
