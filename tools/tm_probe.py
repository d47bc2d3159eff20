"""Compare a forced stage-2 variant with the default one on a config: outputs (max
difference relative to the mass bound of the north star) and per-stage device times
(CUDA-graph replays, warm L2).  Plain text, not a bench line.
Usage: python tools/tm_probe.py VARIANT [cfg[:N]] [s ...]"""
import dataclasses
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1704_07724_b200 import datagen, sparseconv as sc  # noqa: E402
from tools.probe_run import dev_time_us  # noqa: E402


def plan(shp, w, b, force):
    """force: None (default selection), a variant id, or "jit:TY,KL,NW,MINB,CH,STAGES,SLOTS,PIECE"."""
    key = "SC_JIT_FORCE" if isinstance(force, str) else "SC_FORCE_VARIANT"
    val = force[4:] if isinstance(force, str) else force
    old = os.environ.get(key)
    if force is None:
        os.environ.pop(key, None)
    else:
        os.environ[key] = str(val)
    try:
        return sc.SparseConv(w, b, shp.n, shp.c, shp.h, shp.w, shp.stride, shp.pad, shp.groups)
    finally:
        if old is None:
            os.environ.pop(key, None)
        else:
            os.environ[key] = old


def main():
    vid = sys.argv[1] if sys.argv[1].startswith("jit:") else int(sys.argv[1])
    cfg = sys.argv[2] if len(sys.argv) > 2 else "C2"
    sps = [float(v) for v in sys.argv[3:]] or [0.9, 0.95, 0.99]
    cfg, _, nimg = cfg.partition(":")   # "C2:512" overrides the batch; "T2.<layer>" = a paper Table 2 layer
    if cfg.startswith("T2."):
        shp = {s.name: s for s, _ in datagen.table2_shapes(128)}[cfg[3:]]
    else:
        shp = datagen.CONFIGS[cfg]
    if nimg:
        shp = dataclasses.replace(shp, n=int(nimg))
    wn, bn = datagen.weights(shp)
    w, b = torch.from_numpy(wn).cuda(), torch.from_numpy(bn).cuda()
    ref, new = plan(shp, w, b, None), plan(shp, w, b, vid)
    print(f"{cfg}: default {ref.variant} vs forced {new.variant}")
    wabs = torch.from_numpy(np.abs(wn)).cuda()
    for s in sps:
        x = torch.from_numpy(datagen.activations(shp, s)).cuda()
        o1, o2 = ref.forward(x), new.forward(x)
        mass = torch.nn.functional.conv2d(x.abs(), wabs, None, shp.stride, shp.pad, 1, shp.groups)
        err = ((o1 - o2).abs() / (1e-5 * mass + 1e-6)).max().item()
        t = {}
        for name, p in (("default", ref), ("forced", new)):
            out = torch.empty_like(o1)
            t[name] = (dev_time_us(lambda: p.compact(x)), dev_time_us(lambda: p.gather(shp.n, out)),
                       dev_time_us(lambda: p.forward(x, out)))
        print(f"s={s}: max |diff| / (1e-5 mass + 1e-6) = {err:.3f}; finite={bool(torch.isfinite(o2).all())}")
        for name, (c, g, f) in t.items():
            print(f"   {name:8s} compact {c:7.1f} us  gather {g:7.1f} us  forward {f:7.1f} us")


if __name__ == "__main__":
    main()
