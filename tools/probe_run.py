"""Quick GPU probe: FMA-pipe rates and per-stage device times of the sparse
path (and the dense path) per config.  Device times come from CUDA graphs that
hold `reps` back-to-back launches (host launch cost excluded).  Plain text; not
a bench line.  Usage: python tools/probe_run.py [cfg ...]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1704_07724_b200 import datagen, sparseconv as sc  # noqa: E402


def dev_time_us(fn, reps=20):
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        fn()
        s.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s, capture_error_mode="relaxed"):
            for _ in range(reps):
                fn()
        g.replay()
        s.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        g.replay()
        b.record(s)
        b.synchronize()
    return a.elapsed_time(b) * 1e3 / reps


def main():
    cfgs = sys.argv[1:] or ["C2", "C4a", "C3", "C1", "C4b"]
    for kind, name in ((0, "FFMA"), (1, "FFMA2")):
        print(f"probe {name}: {sc.probe_fma(kind):.1f} lane-FMA/clk/SM")
    for cfg in cfgs:
        for s in datagen.CONFIG_SPARSITY[cfg]:
            shp = datagen.CONFIGS[cfg]
            x = torch.from_numpy(datagen.activations(shp, s)).cuda()
            w, b = datagen.weights(shp)
            conv = sc.SparseConv(torch.from_numpy(w).cuda(), torch.from_numpy(b).cuda(), shp.n, shp.c, shp.h,
                                 shp.w, shp.stride, shp.pad, shp.groups)
            out = conv.forward(x)
            t_c = dev_time_us(lambda: conv.compact(x))
            t_g = dev_time_us(lambda: conv.gather(shp.n, out))
            t_f = dev_time_us(lambda: conv.forward(x, out))
            try:
                t_d = dev_time_us(lambda: conv.dense_forward(x, out))
            except sc.SparseConvError:
                t_d = float("nan")
            print(f"{cfg} s={s} variant={conv.variant} compact={t_c:.1f}us gather={t_g:.1f}us "
                  f"forward={t_f:.1f}us dense_tc={t_d:.1f}us")


if __name__ == "__main__":
    main()
