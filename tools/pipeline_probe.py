"""Cross-batch pipelining probe: batch i+1's stage 1 on a low-priority stream overlapping batch
i's stage 2 (two plans = two stage-1 workspaces; stage-2 launches alternate between two
high-priority streams so batch i+1's gather can start in batch i's last wave).  Compares
time per batch against back-to-back sparse_conv_forward on one stream; outputs must be
bit-identical.  Usage: python tools/pipeline_probe.py [cfg] [s] [K]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1704_07724_b200 import datagen, sparseconv as sc  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
s = float(sys.argv[2]) if len(sys.argv) > 2 else 0.95
K = int(sys.argv[3]) if len(sys.argv) > 3 else 24
dev = torch.device("cuda", 0)
shp = datagen.CONFIGS[cfg]
w, b = datagen.weights(shp)
nsets = 6
xs = [torch.from_numpy(datagen.activations(shp, s, seed=i)).to(dev) for i in range(nsets)]
outs = [torch.empty((shp.n, shp.k, shp.ho, shp.wo), device=dev) for _ in range(nsets)]
plans = [sc.SparseConv(torch.from_numpy(w).to(dev), torch.from_numpy(b).to(dev), shp.n, shp.c, shp.h, shp.w,
                       shp.stride, shp.pad, shp.groups) for _ in range(2)]
lo, hi = torch.cuda.Stream.priority_range()
S = torch.cuda.Stream(priority=lo)
G = [torch.cuda.Stream(priority=hi), torch.cuda.Stream(priority=hi)]
cur = torch.cuda.current_stream()
print("variant", plans[0].variant, "priorities", lo, hi, flush=True)


def sequential(k):
    for i in range(k):
        plans[0].forward(xs[i % nsets], outs[i % nsets], stream=cur)


def pipelined(k, gather_streams=2, stage1_low=True):
    ev_g = [torch.cuda.Event(), torch.cuda.Event()]
    ev_s = torch.cuda.Event()
    st1 = S if stage1_low else G[1]
    S.wait_stream(cur)
    for g in G:
        g.wait_stream(cur)
    for i in range(k):
        p = plans[i % 2]
        if i >= 2:
            st1.wait_event(ev_g[i % 2])       # this plan's workspace: its last gather is done
        p.compact(xs[i % nsets], stream=st1)
        ev_s.record(st1)
        g = G[i % gather_streams]
        g.wait_event(ev_s)
        p.gather(shp.n, outs[i % nsets], stream=g)
        ev_g[i % 2].record(g)
    for g in G + [S]:
        cur.wait_stream(g)


def timed(fn, k, reps=5):
    best = []
    for _ in range(reps):
        fn(4)
        torch.cuda.synchronize()
        a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(cur)
        fn(k)
        e.record(cur)
        torch.cuda.synchronize()
        best.append(a.elapsed_time(e) * 1e3 / k)
    return sorted(best)[len(best) // 2]


sequential(nsets)
torch.cuda.synchronize()
ref = [o.clone() for o in outs]
for o in outs:
    o.zero_()
pipelined(nsets)
torch.cuda.synchronize()
same = all(torch.equal(a, b) for a, b in zip(ref, outs))
print("pipelined outputs bit-identical:", same, flush=True)
print(f"sequential           {timed(sequential, K):8.1f} us/batch")
print(f"pipelined            {timed(pipelined, K):8.1f} us/batch")


def library(k, stream=None):
    plans[0].forward_batches([xs[i % nsets] for i in range(k)], [outs[i % nsets] for i in range(k)],
                             stream=stream or cur)


print(f"forward_batches      {timed(library, K):8.1f} us/batch")
plans[0].reserve_batches()
graph_k = 2 * nsets
g = torch.cuda.CUDAGraph()
cap = torch.cuda.Stream()
with torch.cuda.graph(g, stream=cap):
    library(graph_k, cap)
print(f"forward_batches graph of {graph_k} {timed(lambda k: [g.replay() for _ in range(k // graph_k)], graph_k * 2):8.1f} us/batch")
def gather_only(k):  # stage 2 alone, back to back on the two high-priority streams (stage 1 done once)
    for g in G:
        g.wait_stream(cur)
    for i in range(k):
        plans[0].gather(shp.n, outs[i % nsets], stream=G[i % 2])
    for g in G:
        cur.wait_stream(g)


plans[0].compact(xs[0], stream=cur)
print(f"stage 2 only, 2 G    {timed(gather_only, K):8.1f} us/batch")
print(f"pipelined 1 G stream {timed(lambda k: pipelined(k, 1), K):8.1f} us/batch")
print(f"pipelined no prio    {timed(lambda k: pipelined(k, 2, False), K):8.1f} us/batch")
