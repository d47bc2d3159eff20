"""R7 / SURVEY 8c item 7: NaN and +-Inf inputs count as nonzero (IEEE x != 0.0f)
and propagate exactly as in the dense definition (Eq. 1): an output
whose receptive field holds a NaN is NaN, one that sums +Inf and -Inf products
is NaN, one with infinite products of a single sign is that infinity; every
other output meets the usual 1e-5*mass bound.  Sparse path on every BASELINE
config shape (every shipped stage-2 variant kind: k-quads, k-pairs, x-pairs)."""
import numpy as np
import pytest
import torch

import oracle
from lists_check import check_plane_lists
from paper_1704_07724_b200 import datagen

pytestmark = pytest.mark.gpu
DEV = torch.device("cuda:0")


def _inject(x, seed):
    rng = np.random.default_rng(seed)
    flat = x.reshape(-1)
    idx = rng.choice(flat.size, size=6, replace=False)
    flat[idx[:2]] = np.nan
    flat[idx[2:4]] = np.inf
    flat[idx[4:]] = -np.inf
    return x


def _compare(got, ref, mass):
    nan_ref = np.isnan(ref)
    assert np.array_equal(np.isnan(got), nan_ref), "NaN pattern differs from the dense definition"
    inf_ref = np.isinf(ref)
    assert np.array_equal(np.isinf(got), inf_ref), "Inf pattern differs"
    assert np.array_equal(np.sign(got[inf_ref]), np.sign(ref[inf_ref])), "Inf signs differ"
    fin = np.isfinite(ref)
    assert np.all(np.abs(got[fin] - ref[fin]) <= oracle.tolerance_sparse(mass[fin]))
    return int(nan_ref.sum()), int(inf_ref.sum())


@pytest.mark.parametrize("cfg", ["C1", "C2", "C3", "C4a", "C4b"])
def test_nan_inf_propagate_like_the_definition(cfg):
    from paper_1704_07724_b200 import sparseconv as sc
    shp = datagen.CONFIGS[cfg].with_batch(2)
    s = datagen.CONFIG_SPARSITY[cfg][0]
    x = _inject(datagen.activations(shp, s, seed=9), 9)
    w, b = datagen.weights(shp, seed=9)
    conv = sc.SparseConv(torch.from_numpy(w).to(DEV), torch.from_numpy(b).to(DEV), shp.n, shp.c, shp.h, shp.w,
                         shp.stride, shp.pad, shp.groups)
    got = conv.forward(torch.from_numpy(x).to(DEV)).cpu().numpy().astype(np.float64)
    check_plane_lists(conv, x, shp.n)                      # NaN/Inf are listed with their bits
    ref, mass = oracle.conv_fp64(x, w, b, shp.stride, shp.pad, shp.groups)
    nans, infs = _compare(got, ref, mass)
    assert nans > 0                                        # the case exercises propagation
