"""Backward shape sweep (robustness, not a CI test): random shapes the backward
supports (1x1 / 3x3 / 5x5, stride <= 2, planes of <= 1024 elements and <= 31 rows),
random sparsity, random batch below the plan's -- each checked like
tests/test_gpu_backward.py: dW / dbias / dz within gamma_m * mass of
oracle.conv_backward_fp64 (m = the definition's term count), exact zeros of dz
where the input is zero, and integer data bit-exact.
Usage: python tools/bwd_fuzz.py [shapes] [seed]"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import oracle  # noqa: E402
from paper_1704_07724_b200 import datagen, sparseconv as sc  # noqa: E402
from test_gpu_backward import check_all, dout_for  # noqa: E402

DEV = torch.device("cuda:0")


def shapes(count, seed):
    rng = np.random.default_rng(seed)
    out = []
    while len(out) < count:
        r = int(rng.choice([1, 3, 5]))
        stride = int(rng.choice([1, 1, 2])) if r > 1 else 1
        pad = int(rng.integers(0, r // 2 + 1))
        h, w = int(rng.integers(max(1, r - 2 * pad), 32)), int(rng.integers(max(1, r - 2 * pad), 33))
        if h * w > 1024 or h > 31:
            continue
        groups = int(rng.choice([1, 1, 2]))
        c = groups * int(rng.integers(1, 40))
        k = groups * int(rng.integers(1, 150))
        n = int(rng.integers(1, 9))
        out.append(datagen.ConvShape(f"bwdfuzz{seed}_{len(out)}", 4000 + len(out), n, c, h, w, k, r, r, stride, pad,
                                     groups))
    return out


def main():
    count = int(sys.argv[1]) if len(sys.argv) > 1 else 60
    seed = int(sys.argv[2]) if len(sys.argv) > 2 else 0
    fails = 0
    for shp in shapes(count, seed):
        s = float(np.random.default_rng(shp.config_id).choice([0.0, 0.5, 0.9, 0.97]))
        n = max(1, shp.n - 1)  # ragged: n of an n+1 plan when possible
        try:
            x = datagen.activations(shp, s, seed=shp.config_id)[:n]
            w, b = datagen.weights(shp, seed=shp.config_id)
            d = dout_for(shp, n, shp.config_id)
            conv = sc.SparseConv(torch.from_numpy(w).to(DEV), torch.from_numpy(b).to(DEV), shp.n, shp.c, shp.h,
                                 shp.w, shp.stride, shp.pad, shp.groups)
            dw, db, dz = conv.backward(torch.from_numpy(np.ascontiguousarray(x)).to(DEV), torch.from_numpy(d).to(DEV))
            torch.cuda.synchronize()
            got = tuple(t.cpu().numpy() for t in (dw, db, dz))
            ref = oracle.conv_backward_fp64(x, w, d, shp.stride, shp.pad, shp.groups)
            check_all(got, ref, shp, n, shp.n, d)
            assert np.all(got[2][x == 0] == 0), "dz not zero where the input is zero"
            xi, wi, _ = datagen.integer_case(shp.with_batch(n), sparsity=0.6)
            di = dout_for(shp, n, shp.config_id + 1, integer=True)
            convi = sc.SparseConv(torch.from_numpy(wi).to(DEV), None, shp.n, shp.c, shp.h, shp.w, shp.stride,
                                  shp.pad, shp.groups)
            dwi, _, dzi = convi.backward(torch.from_numpy(xi).to(DEV), torch.from_numpy(di).to(DEV))
            torch.cuda.synchronize()
            refi = oracle.conv_backward_fp64(xi, wi, di, shp.stride, shp.pad, shp.groups, want_mass=False)
            assert np.array_equal(dwi.cpu().numpy().astype(np.float64), refi["dw"]), "integer dW"
            assert np.array_equal(dzi.cpu().numpy().astype(np.float64), refi["dz"]), "integer dz"
            print(f"ok   {shp} n={n} s={s}", flush=True)
        except sc.SparseConvError as e:
            if e.status == 3:
                print(f"skip {shp}: {e}", flush=True)
                continue
            fails += 1
            print(f"FAIL {shp} n={n} s={s}: {e}", flush=True)
        except AssertionError as e:
            fails += 1
            print(f"FAIL {shp} n={n} s={s}: {e}", flush=True)
    print(f"{count - fails}/{count} passed (skips counted as passed)")
    return 1 if fails else 0


if __name__ == "__main__":
    sys.exit(main())
