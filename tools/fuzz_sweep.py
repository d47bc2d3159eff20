"""Extended shape sweep (robustness, not a CI test): random shapes beyond
tests/test_gpu_fuzz.py -- more seeds, larger channel and filter counts, batches
that make multi-wave stage-2 grids -- each checked like the fuzz test: stage-1
lists bit-exact against the oracle, streams against the test-side adapter,
sparse outputs within 1e-5*mass + 1e-6, integer data bit-exact.
Usage: python tools/fuzz_sweep.py [seeds] [shapes per seed] [first seed] [wide]
("wide": a quarter of the shapes are 1x1 layers with 150-520 filters per group)"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import oracle  # noqa: E402
from lists_check import check_plane_lists, check_streams  # noqa: E402
from paper_1704_07724_b200 import datagen, sparseconv as sc  # noqa: E402

DEV = torch.device("cuda:0")
WIDE = len(sys.argv) > 4 and sys.argv[4] == "wide"


def shapes(seed, count):
    rng = np.random.default_rng(seed)
    out = []
    for i in range(count):
        groups = int(rng.choice([1, 1, 1, 2, 4]))
        c = groups * int(rng.integers(1, 40))
        k = groups * int(rng.integers(1, 100))
        h, w = int(rng.integers(1, 34)), int(rng.integers(1, 34))
        stride = int(rng.choice([1, 1, 1, 2, 3]))
        pad = int(rng.integers(0, 4))
        r = int(rng.integers(1, min(7, h + 2 * pad) + 1))
        s = int(rng.integers(1, min(7, w + 2 * pad) + 1))
        n = int(rng.choice([1, 3, 8, 40]))
        if WIDE and rng.random() < 0.25:  # 1x1 with many filters: the KL = 6 / 8 rule (sc_internal.h wide_1x1_kl)
            r = s = stride = 1
            pad = 0
            k = groups * int(rng.integers(150, 521))
        out.append(datagen.ConvShape(f"sweep{seed}_{i}", 2000 + 100 * seed + i, n, c, h, w, k, r, s, stride, pad,
                                     groups))
    return out


def check(shp, sparsity):
    x = datagen.activations(shp, sparsity, seed=7)
    w, b = datagen.weights(shp, seed=7)
    conv = sc.SparseConv(torch.from_numpy(w).to(DEV), torch.from_numpy(b).to(DEV), shp.n, shp.c, shp.h, shp.w,
                         shp.stride, shp.pad, shp.groups)
    out = conv.forward(torch.from_numpy(x).to(DEV)).cpu().numpy()
    kept = check_plane_lists(conv, x, shp.n)
    check_streams(conv, x, shp.n)
    ref, mass = oracle.conv_fp64(x, w, b, shp.stride, shp.pad, shp.groups)
    ratio = float(np.max(np.abs(out - ref) / oracle.tolerance_sparse(mass)))
    assert ratio <= 1.0, f"sparse err/tol {ratio}"
    xi, wi, bi = datagen.integer_case(shp, sparsity=0.7, seed=7)
    convi = sc.SparseConv(torch.from_numpy(wi).to(DEV), torch.from_numpy(bi).to(DEV), shp.n, shp.c, shp.h, shp.w,
                          shp.stride, shp.pad, shp.groups)
    oi = convi.forward(torch.from_numpy(xi).to(DEV)).cpu().numpy().astype(np.float64)
    refi, _ = oracle.conv_fp64(xi, wi, bi, shp.stride, shp.pad, shp.groups)
    assert np.array_equal(oi, refi), "integer data not bit-exact"
    return conv.variant[1], kept, ratio


def main():
    seeds = int(sys.argv[1]) if len(sys.argv) > 1 else 4
    count = int(sys.argv[2]) if len(sys.argv) > 2 else 30
    first = int(sys.argv[3]) if len(sys.argv) > 3 else 0  # first seed
    fails = 0
    total = 0
    for seed in range(first, first + seeds):
        for shp in shapes(seed, count):
            for s in (0.95, 0.5):
                total += 1
                try:
                    v, kept, ratio = check(shp, s)
                    print(f"ok   {shp.name} s={s} {shp} variant={v} lists={'plane' if kept else 'streamwise'} "
                          f"err/tol={ratio:.3f}", flush=True)
                except Exception as e:  # report and continue
                    fails += 1
                    print(f"FAIL {shp.name} s={s} {shp}: {type(e).__name__}: {str(e)[:200]}", flush=True)
    print(f"{total - fails}/{total} passed", flush=True)
    return 1 if fails else 0


if __name__ == "__main__":
    sys.exit(main())
