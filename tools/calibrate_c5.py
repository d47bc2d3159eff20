"""Write paper_1704_07724_b200/c5_bias_shift.json (reading R13).

C5 (BASELINE.json configs[4]) asks for "bias shifted negative to hold
s ~ 0.95" on the conv3->conv4->conv5 chain.  Reading R13: per layer l whose
output feeds a ReLU (conv3, conv4), q_l = 95th percentile of the
pre-activation (conv + N(0,0.01^2) bias) over a calibration subset (the first
16 images), computed with the fp64 ORACLE, chained; the layer's bias becomes
bias - q_l.  conv5 has no downstream ReLU and is unshifted.

Calls only oracle/ and the seeded generators (no CUDA path).
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
from paper_1704_07724_b200 import datagen  # noqa: E402


def main(n_cal=16, seed=0):
    shapes = datagen.C5_LAYERS
    x = datagen.activations(shapes[0].with_batch(n_cal), datagen.C5_FIRST_SPARSITY, seed)
    shifts = {}
    for li, shp in enumerate(shapes):
        w, b = datagen.weights(shp, seed)
        pre, _ = oracle.conv_fp64(x, w, b, shp.stride, shp.pad, shp.groups, want_mass=False)
        if li < 2:
            q = float(np.percentile(pre, 95.0))
            shifts[shp.name] = q
            b_shift = (b - np.float32(q)).astype(np.float32)
            pre, _ = oracle.conv_fp64(x, w, b_shift, shp.stride, shp.pad, shp.groups, want_mass=False)
            x = oracle.relu(pre.astype(np.float32))
            print(f"{shp.name}: q={q:.6g}  next-input sparsity={oracle.sparsity(x):.4f}")
        else:
            shifts[shp.name] = 0.0
    out = os.path.join(ROOT, "paper_1704_07724_b200", "c5_bias_shift.json")
    with open(out, "w") as f:
        json.dump(shifts, f, indent=1)
        f.write("\n")
    print("wrote", out, shifts)


if __name__ == "__main__":
    main()
