"""GPU parity of the sparse backward (sparse_conv_backward, SURVEY 8f row f4,
DESIGN.md R19-R20) against oracle.conv_backward_fp64.

Bars:
* integer-valued data: bit-exact (every partial sum is an integer < 2^24);
* random data: |gpu - oracle| <= gamma_m * mass + 1e-30 per element,
  gamma_m = m*u / (1 - m*u), u = 2^-24, the bound for any evaluation order
  of an m-term fp32 sum of products, with m the term count of the definition
  (R19): wgrad and dbias m = N*Ho*Wo, dgrad m = Kg*R*S."""
import numpy as np
import pytest
import torch

import oracle
from paper_1704_07724_b200 import datagen

pytestmark = pytest.mark.gpu
DEV = torch.device("cuda:0")
U = 2.0 ** -24


@pytest.fixture(scope="module")
def sc():
    from paper_1704_07724_b200 import sparseconv
    sparseconv.lib()
    return sparseconv


def make_conv(sc, shp, w, b=None, max_batch=None):
    return sc.SparseConv(torch.from_numpy(w).to(DEV), None if b is None else torch.from_numpy(b).to(DEV),
                         max_batch or shp.n, shp.c, shp.h, shp.w, shp.stride, shp.pad, shp.groups)


def gamma(m):
    return m * U / (1 - m * U)


def chains(shp, n, max_batch=None):
    """Term counts of the three sums as the definitions state them (R19):
    dW[k,c,r,t] sums over (n, y, x): N*Ho*Wo terms; dz[n,c,i,j] over (k, r, t) of
    the group: Kg*R*S terms; dbias[k] over (n, y, x): N*Ho*Wo terms.  Any
    evaluation order of an m-term sum of products (FMA or not) is within
    gamma_m * sum|terms| of the exact value (Higham, Accuracy and Stability,
    Sec. 3.1), so the bound is fixed by the problem, not by the kernel."""
    howo = shp.ho * shp.wo
    return n * howo, (shp.k // shp.groups) * shp.r * shp.s, n * howo


def dout_for(shp, n, seed, integer=False):
    rng = np.random.default_rng(seed)
    if integer:
        return rng.integers(-4, 5, (n, shp.k, shp.ho, shp.wo)).astype(np.float32)
    return rng.standard_normal((n, shp.k, shp.ho, shp.wo)).astype(np.float32)


def run_bwd(conv, x, d, **kw):
    dw, db, dz = conv.backward(torch.from_numpy(x).to(DEV), torch.from_numpy(d).to(DEV), **kw)
    torch.cuda.synchronize()
    return tuple(None if t is None else t.cpu().numpy() for t in (dw, db, dz))


def check_all(got, ref, shp, n, max_batch, d):
    dw, db, dz = got
    m_w, m_d, m_b = chains(shp, n, max_batch)
    if dw is not None:
        err = np.abs(dw - ref["dw"])
        tol = gamma(m_w) * ref["dw_mass"] + 1e-30
        assert np.all(err <= tol), f"dw: max err/tol {(err / tol).max():.3f}"
    if db is not None:
        tol = gamma(m_b) * np.abs(d.astype(np.float64)).sum(axis=(0, 2, 3)) + 1e-30
        assert np.all(np.abs(db - ref["dbias"]) <= tol), "dbias"
    if dz is not None:
        err = np.abs(dz - ref["dz"])
        tol = gamma(m_d) * ref["dz_mass"] + 1e-30
        assert np.all(err <= tol), f"dz: max err/tol {(err / tol).max():.3f}"


@pytest.mark.parametrize("cfg", ["C1", "C2", "C3", "C4a", "C4b"])
@pytest.mark.parametrize("s", [0.0, 0.9, 0.99])
def test_backward_small_batch(sc, cfg, s):
    shp = datagen.CONFIGS[cfg].with_batch(3)
    x = datagen.activations(shp, s if cfg != "C3" or s == 0.0 else "channel", seed=21)
    w, b = datagen.weights(shp, seed=21)
    d = dout_for(shp, 3, 21)
    conv = make_conv(sc, shp, w, b, max_batch=4)  # ragged: n=3 of a 4-image plan
    got = run_bwd(conv, x, d)
    ref = oracle.conv_backward_fp64(x, w, d, shp.stride, shp.pad, shp.groups)
    check_all(got, ref, shp, 3, 4, d)
    assert np.all(got[2][x == 0] == 0)  # through the ReLU: exact zeros where in == 0


@pytest.mark.parametrize("cfg", ["C1", "C2", "C3", "C4a", "C4b"])
def test_backward_integer_bitexact(sc, cfg):
    shp = datagen.CONFIGS[cfg].with_batch(2)
    x, w, _ = datagen.integer_case(shp, sparsity=0.7)
    d = dout_for(shp, 2, 5, integer=True)
    conv = make_conv(sc, shp, w)
    dw, db, dz = run_bwd(conv, x, d)
    ref = oracle.conv_backward_fp64(x, w, d, shp.stride, shp.pad, shp.groups, want_mass=False)
    assert np.array_equal(dw.astype(np.float64), ref["dw"])
    assert np.array_equal(db.astype(np.float64), ref["dbias"])
    assert np.array_equal(dz.astype(np.float64), ref["dz"])


def test_backward_table2_shapes(sc):
    for shp, s in datagen.table2_shapes(n=2):
        x = datagen.activations(shp, s)
        w, b = datagen.weights(shp)
        d = dout_for(shp, 2, 8)
        conv = make_conv(sc, shp, w, b)
        got = run_bwd(conv, x, d)
        ref = oracle.conv_backward_fp64(x, w, d, shp.stride, shp.pad, shp.groups)
        check_all(got, ref, shp, 2, 2, d)
        xi, wi, _ = datagen.integer_case(shp, sparsity=0.5)
        di = dout_for(shp, 2, 9, integer=True)
        conv = make_conv(sc, shp, wi)
        dw, db, dz = run_bwd(conv, xi, di)
        ref = oracle.conv_backward_fp64(xi, wi, di, shp.stride, shp.pad, shp.groups, want_mass=False)
        assert np.array_equal(dw.astype(np.float64), ref["dw"]), shp.name
        assert np.array_equal(dz.astype(np.float64), ref["dz"]), shp.name


def test_backward_edge_cases(sc):
    shp = datagen.C2.with_batch(2)
    w, b = datagen.weights(shp, seed=4)
    d = dout_for(shp, 2, 4)
    conv = make_conv(sc, shp, w, b)
    z = np.zeros((2, shp.c, shp.h, shp.w), np.float32)
    dw, db, dz = run_bwd(conv, z, d)
    assert not dw.any() and not dz.any()
    # outputs are independent and nullable
    x = datagen.activations(shp, 0.95, seed=4)
    full = run_bwd(conv, x, d)
    only_dz = run_bwd(conv, x, d, want_dw=False, want_dbias=False)
    only_dw = run_bwd(conv, x, d, want_dz=False, want_dbias=False)
    assert only_dz[0] is None and only_dw[2] is None
    assert np.array_equal(only_dz[2], full[2]) and np.array_equal(only_dw[0], full[0])
    # one image of a two-image plan
    got = run_bwd(conv, x[:1], d[:1])
    ref = oracle.conv_backward_fp64(x[:1], w, d[:1], 1, 1, 1)
    check_all(got, ref, shp, 1, 2, d[:1])
    # deterministic: a second call is bit-identical
    again = run_bwd(conv, x, d)
    for a_, b_ in zip(full, again):
        assert np.array_equal(a_, b_)


@pytest.mark.parametrize("shp", [
    datagen.ConvShape("plane1600", 99, 2, 4, 40, 40, 8, 3, 3, 1, 1, 1),  # H*W > 1024: no plane-major lists
    datagen.ConvShape("k7", 99, 2, 4, 8, 8, 8, 7, 7, 1, 3, 1),           # 7x7 is not instantiated
])
def test_backward_unsupported_shape(sc, shp):
    w, _ = datagen.weights(shp)
    conv = make_conv(sc, shp, w)
    x = torch.zeros((2, shp.c, shp.h, shp.w), device=DEV)
    d = torch.zeros((2, shp.k, shp.ho, shp.wo), device=DEV)
    with pytest.raises(sc.SparseConvError):
        conv.backward(x, d)


@pytest.mark.parametrize("cfg,s", [("C2", 0.95), ("C4a", 0.9), ("C3", "channel")])
def test_backward_full_config_sampled(sc, cfg, s):
    """BASELINE sizes in the bench's launch configuration; the oracle checks
    dw on a channel x filter slice (dw[k,c] depends only on in[:,c], dout[:,k])
    and dz on sampled images (dz[n] depends only on image n)."""
    shp = datagen.CONFIGS[cfg]
    n = shp.n
    x = datagen.activations(shp, s)
    w, b = datagen.weights(shp)
    d = dout_for(shp, n, 31)
    conv = make_conv(sc, shp, w, b)
    dw, db, dz = run_bwd(conv, x, d)
    m_w, m_d, m_b = chains(shp, n, n)
    cg, kg = shp.c // shp.groups, shp.k // shp.groups
    for g in range(shp.groups):
        cs = np.arange(g * cg, g * cg + min(cg, 8))
        ks = np.arange(g * kg, g * kg + min(kg, 8))
        ref = oracle.conv_backward_fp64(x[:, cs], w[ks][:, :len(cs)], d[:, ks], shp.stride, shp.pad, 1)
        got = dw[ks][:, cs - g * cg]
        tol = gamma(m_w) * ref["dw_mass"] + 1e-30
        assert np.all(np.abs(got - ref["dw"]) <= tol), f"dw slice group {g}"
    for i0 in (0, n // 2, n - 1):
        ref = oracle.conv_backward_fp64(x[i0:i0 + 1], w, d[i0:i0 + 1], shp.stride, shp.pad, shp.groups)
        tol = gamma(m_d) * ref["dz_mass"] + 1e-30
        assert np.all(np.abs(dz[i0:i0 + 1] - ref["dz"]) <= tol), f"dz image {i0}"
    # dbias depends on dout only: the oracle on a one-channel, one-group slice
    ref = oracle.conv_backward_fp64(x[:, :1], w[:, :1], d, shp.stride, shp.pad, 1, want_mass=False)
    tolb = gamma(m_b) * np.abs(d.astype(np.float64)).sum(axis=(0, 2, 3)) + 1e-30
    assert np.all(np.abs(db - ref["dbias"]) <= tolb)


@pytest.mark.parametrize("variant", ["3,3,11,1,8,4,3,254", 21, "7,1,11,1,16,4,3,254", "7,2,7,1,8,4,3,254"])
def test_backward_with_every_weight_packing(sc, variant, monkeypatch):
    """The backward reads the forward's packed weights: k-blocks of 32*KL with KL = 3 (permuted
    pair/single layout), 4 (V21), 1 and 2 (run-time generated tilings, SC_JIT_FORCE) must all
    give the same gradients."""
    if isinstance(variant, str):
        monkeypatch.setenv("SC_JIT_FORCE", variant)
    else:
        monkeypatch.setenv("SC_FORCE_VARIANT", str(variant))
    shp = datagen.C2.with_batch(2)
    x = datagen.activations(shp, 0.9, seed=12)
    w, b = datagen.weights(shp, seed=12)
    d = dout_for(shp, 2, 12)
    conv = make_conv(sc, shp, w, b)
    assert conv.variant[0] == (-1 if isinstance(variant, str) else variant)
    got = run_bwd(conv, x, d)
    ref = oracle.conv_backward_fp64(x, w, d, shp.stride, shp.pad, shp.groups)
    check_all(got, ref, shp, 2, 2, d)
