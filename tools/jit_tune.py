"""Sweep run-time generated stage-2 variants for one config (SC_JIT_FORCE knob):
python tools/jit_tune.py C2 0.95 [quick]
Prints one line per parameter set: gather time (graph, warm L2), max err/tol on two
oracle images, sorted by time at the end."""
import itertools
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
from paper_1704_07724_b200 import datagen, sparseconv as sc  # noqa: E402
from tools.probe_run import dev_time_us  # noqa: E402

cfg, s = sys.argv[1], (sys.argv[2] if sys.argv[2] == "channel" else float(sys.argv[2]))
quick = len(sys.argv) > 3
if cfg.startswith("T2:"):  # a paper Table 2 layer by name, N=128
    shp = {t.name: t for t, _ in datagen.table2_shapes(n=128)}[cfg[3:]]
elif cfg.startswith("C5."):  # a layer of the C5 chain (i.i.d. input at s), N from TUNE_N (default 256)
    shp = datagen.C5_LAYERS[int(cfg[3:])].with_batch(int(os.environ.get("TUNE_N", "256")))
else:
    shp = datagen.CONFIGS[cfg]
w, b = datagen.weights(shp)
xh = datagen.activations(shp, s)
x = torch.from_numpy(xh).cuda()
refs = {i: oracle.conv_fp64(xh[i:i + 1], w, b, shp.stride, shp.pad, shp.groups) for i in (0, shp.n - 1)}
out = torch.empty((shp.n, shp.k, shp.ho, shp.wo), device="cuda")

grid = [(2, 4), (1, 4), (2, 2), (3, 2), (4, 2), (2, 3), (3, 3)]
if (shp.k // shp.groups <= 64 or os.environ.get("TUNE_XPAIR")) and shp.stride == 1 and shp.s >= 2:  # x-pair tiles
    grid += [(2, 1), (3, 1), (4, 1), (5, 1), (6, 1), (7, 1), (1, 1)]
grid += [(5, 2), (6, 2), (7, 2), (5, 4), (4, 4)]
grid = [(ty, kl) for ty, kl in grid if ty <= shp.ho]
if os.environ.get("TUNE_ONLY_XPAIR"):
    grid = [(ty, kl) for ty, kl in grid if kl == 1]
nws = [11, 9] if not quick else [11]
chs = [16, 32, 8] if not quick else [16]
stages = [2, 3]
slots = [3, 4, 2]
pieces = [254, 510, 126]


def env_list(name, default):  # e.g. TUNE_CHS="8,12,16"
    v = os.environ.get(name)
    return [int(t) for t in v.split(",")] if v else default


if os.environ.get("TUNE_GRID"):  # "2:4,1:4" = (TY, KL) pairs
    grid = [tuple(int(u) for u in t.split(":")) for t in os.environ["TUNE_GRID"].split(",")]
nws, chs, stages = env_list("TUNE_NWS", nws), env_list("TUNE_CHS", chs), env_list("TUNE_STAGES", stages)
slots, pieces = env_list("TUNE_SLOTS", slots), env_list("TUNE_PIECES", pieces)
full = cfg.startswith("T2:") or bool(os.environ.get("TUNE_FULL"))  # time the whole forward (the tile height changes stage 1 too)
pipe = bool(os.environ.get("TUNE_PIPE"))  # time per batch of 12 batches through forward_batches (pipelined steps)
out2 = torch.empty_like(out)


def pipe_time(conv):
    xs, outs = [x] * 12, [out, out2] * 6  # batches b, b+2 share a stage-2 stream, so an output buffer
    conv.reserve_batches()
    return dev_time_us(lambda: conv.forward_batches(xs, outs), reps=5) / 12
os.environ.pop("SC_JIT_FORCE", None)
base = sc.SparseConv(torch.from_numpy(w).cuda(), torch.from_numpy(b).cuda(), shp.n, shp.c, shp.h, shp.w,
                     shp.stride, shp.pad, shp.groups)
tb = pipe_time(base) if pipe else (dev_time_us(lambda: base.forward(x, out), reps=10) if full else None)
print("shipped", base.variant, f"{'pipelined' if pipe else 'forward'} {tb:.1f} us" if tb else "", flush=True)
del base
res = []
for (ty, kl), nw, ch, st, sl, pc in itertools.product(grid, nws, chs, stages, slots, pieces):
    os.environ["SC_JIT_FORCE"] = f"{ty},{kl},{nw},1,{ch},{st},{sl},{pc}"
    try:
        conv = sc.SparseConv(torch.from_numpy(w).cuda(), torch.from_numpy(b).cuda(), shp.n, shp.c, shp.h, shp.w,
                             shp.stride, shp.pad, shp.groups)
    except sc.SparseConvError as e:
        print(os.environ["SC_JIT_FORCE"], "create failed", e, flush=True)
        continue
    if conv.variant[0] != -1:
        continue  # compile failed (e.g. shared memory) -> generic
    conv.forward(x, out)
    torch.cuda.synchronize()
    o = out.cpu().numpy()
    worst = max(float((np.abs(o[i:i + 1] - r) / oracle.tolerance_sparse(m)).max()) for i, (r, m) in refs.items())
    if pipe:
        t = pipe_time(conv)
    elif full:
        t = dev_time_us(lambda: conv.forward(x, out), reps=10)
    else:
        conv.compact(x)
        t = dev_time_us(lambda: conv.gather(shp.n, out), reps=10)
    res.append((t, os.environ["SC_JIT_FORCE"], worst, conv.variant[1]))
    print(f"{os.environ['SC_JIT_FORCE']:28s} gather {t:8.1f} us  err/tol {worst:.3f}  {conv.variant[1]}", flush=True)
    del conv
os.environ.pop("SC_JIT_FORCE", None)
print("---- best")
for t, p, wv, n in sorted(res)[:12]:
    print(f"{p:28s} {t:8.1f} us err/tol {wv:.3f}")
