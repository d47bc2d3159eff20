"""GPU parity of the dense comparison path (dense_conv_forward: tcgen05 TF32
implicit GEMM) against the CPU oracle.

Bars (reading R10): operands are rounded to TF32 (cvt.rna), so the
north star's 1e-5 bound is replaced by |gpu - oracle| <= 2^-9 * mass + 1e-6;
integer-valued data is exact in TF32 and fp32, so it must match bit for bit."""
import numpy as np
import pytest
import torch

import oracle
from paper_1704_07724_b200 import datagen

pytestmark = pytest.mark.gpu
DEV = torch.device("cuda:0")


@pytest.fixture(scope="module")
def sc():
    from paper_1704_07724_b200 import sparseconv
    sparseconv.lib()
    return sparseconv


def make_conv(sc, shp, w, b, relu=False, max_batch=None):
    return sc.SparseConv(torch.from_numpy(w).to(DEV), None if b is None else torch.from_numpy(b).to(DEV),
                         max_batch or shp.n, shp.c, shp.h, shp.w, shp.stride, shp.pad, shp.groups, fuse_relu=relu)


def check_dense(got, x, w, b, shp, relu=False, images=None):
    images = range(x.shape[0]) if images is None else images
    for i0 in images:
        ref, mass = oracle.conv_fp64(x[i0:i0 + 1], w, b, shp.stride, shp.pad, shp.groups)
        if relu:
            ref = np.maximum(ref, 0.0)
        err = np.abs(got[i0:i0 + 1].astype(np.float64) - ref)
        tol = oracle.tolerance_dense_tf32(mass)
        assert np.all(err <= tol), f"image {i0}: max err/tol {(err / tol).max():.3f}"


@pytest.mark.parametrize("cfg", ["C1", "C2", "C3", "C4a", "C4b"])
@pytest.mark.parametrize("s", [0.0, 0.95])
def test_dense_small_batch(sc, cfg, s):
    shp = datagen.CONFIGS[cfg].with_batch(3)
    x = datagen.activations(shp, s if cfg != "C3" or s == 0.0 else "channel", seed=7)
    w, b = datagen.weights(shp, seed=7)
    conv = make_conv(sc, shp, w, b, max_batch=4)
    out = conv.dense_forward(torch.from_numpy(x).to(DEV))
    torch.cuda.synchronize()
    check_dense(out.cpu().numpy(), x, w, b, shp)


@pytest.mark.parametrize("cfg", ["C1", "C2", "C3", "C4a", "C4b"])
def test_dense_integer_bitexact(sc, cfg):
    shp = datagen.CONFIGS[cfg].with_batch(3)
    x, w, b = datagen.integer_case(shp, sparsity=0.5)
    conv = make_conv(sc, shp, w, b)
    out = conv.dense_forward(torch.from_numpy(x).to(DEV)).cpu().numpy()
    ref, _ = oracle.conv_fp64(x, w, b, shp.stride, shp.pad, shp.groups)
    assert np.array_equal(out.astype(np.float64), ref)


def test_dense_table2_shapes(sc):
    for shp, s in datagen.table2_shapes(n=2):
        x = datagen.activations(shp, s)
        w, b = datagen.weights(shp)
        conv = make_conv(sc, shp, w, b)
        out = conv.dense_forward(torch.from_numpy(x).to(DEV)).cpu().numpy()
        check_dense(out, x, w, b, shp)
        xi, wi, bi = datagen.integer_case(shp, sparsity=0.5)
        conv = make_conv(sc, shp, wi, bi)
        out = conv.dense_forward(torch.from_numpy(xi).to(DEV)).cpu().numpy()
        ref, _ = oracle.conv_fp64(xi, wi, bi, shp.stride, shp.pad, shp.groups)
        assert np.array_equal(out.astype(np.float64), ref), shp.name


@pytest.mark.parametrize("cfg,s", [("C2", 0.95), ("C3", "channel"), ("C4a", 0.9)])
def test_dense_full_config_sampled(sc, cfg, s):
    shp = datagen.CONFIGS[cfg]
    x = datagen.activations(shp, s)
    w, b = datagen.weights(shp)
    conv = make_conv(sc, shp, w, b)
    out = conv.dense_forward(torch.from_numpy(x).to(DEV)).cpu().numpy()
    check_dense(out, x, w, b, shp, images=[0, shp.n // 2, shp.n - 1])


def test_dense_fused_relu_and_ragged_batch(sc):
    shp = datagen.C2.with_batch(5)
    x = datagen.activations(shp, 0.9)
    w, b = datagen.weights(shp)
    conv = make_conv(sc, shp, w, b, relu=True, max_batch=9)
    out = conv.dense_forward(torch.from_numpy(x).to(DEV)).cpu().numpy()
    assert out.min() >= 0
    check_dense(out, x, w, b, shp, relu=True)


def test_dense_and_sparse_agree_on_integers(sc):
    shp = datagen.C2.with_batch(2)
    x, w, b = datagen.integer_case(shp, sparsity=0.9)
    conv = make_conv(sc, shp, w, b)
    xd = torch.from_numpy(x).to(DEV)
    assert torch.equal(conv.forward(xd), conv.dense_forward(xd))
