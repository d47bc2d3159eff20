"""Pins of oracle.conv_backward_fp64 (R19-R20)
against things other than itself:

* exact rational brute force in the paper's input-stationary (scatter) order
  (ISC: each nonzero input times every weight it meets) -- a different
  loop nest from the oracle's output-stationary definition;
* torch autograd in float64 (conv2d backward: an independent library routine),
  the input gradient masked by the ReLU derivative (Eq. 2);
* Euler/adjoint identities from the linearity of Eq. 1 in W and in `in`,
  evaluated with the (separately pinned) forward oracle:
  sum dout*(conv(in,W)) == sum dw*W == sum dz*in;
* closed forms: a 1x1 stride-1 convolution is a matmul per group, so
  dw = dout_g @ in_g^T and dz = mask * (W_g^T @ dout_g);
* special cases: all-zero input -> dw = 0, dz = 0; dbias = sum of dout."""
import fractions

import numpy as np
import pytest
import torch

import oracle


def _case(seed, integer=False):
    rng = np.random.default_rng(2000 + seed)
    groups = int(rng.integers(1, 3))
    n = int(rng.integers(1, 3))
    c = groups * int(rng.integers(1, 3))
    k = groups * int(rng.integers(1, 3))
    h, ww = int(rng.integers(1, 6)), int(rng.integers(1, 6))
    stride = int(rng.integers(1, 3))
    pad = int(rng.integers(0, 3))
    r = int(rng.integers(1, min(4, h + 2 * pad) + 1))
    s = int(rng.integers(1, min(4, ww + 2 * pad) + 1))
    ho, wo = (h + 2 * pad - r) // stride + 1, (ww + 2 * pad - s) // stride + 1
    mask = rng.random((n, c, h, ww)) < 0.6
    if integer:
        x = np.where(mask, rng.integers(1, 8, (n, c, h, ww)), 0).astype(np.float32)
        w = rng.integers(-8, 9, (k, c // groups, r, s)).astype(np.float32)
        d = rng.integers(-8, 9, (n, k, ho, wo)).astype(np.float32)
    else:
        x = np.where(mask, np.abs(rng.standard_normal((n, c, h, ww))), 0).astype(np.float32)
        w = rng.standard_normal((k, c // groups, r, s)).astype(np.float32)
        d = rng.standard_normal((n, k, ho, wo)).astype(np.float32)
    return x, w, d, stride, pad, groups


def brute_scatter_backward(x, w, d, stride, pad, groups):
    """Exact rationals, input-stationary: for every nonzero input and every
    weight it meets (output index (i+P-r)/T integral and in range)."""
    n, c, h, ww = x.shape
    k, cg, r, s = w.shape
    _, _, ho, wo = d.shape
    kg = k // groups
    F = fractions.Fraction
    dw = np.empty(w.shape, object)
    dw[...] = F(0)
    dz = np.empty(x.shape, object)
    dz[...] = F(0)
    for nn, cc, i, j in zip(*np.nonzero(x)):
        v = F(float(x[nn, cc, i, j]))
        g, cl = cc // cg, cc % cg
        for kk in range(g * kg, (g + 1) * kg):
            for rr in range(r):
                if (i + pad - rr) % stride or i + pad - rr < 0:
                    continue
                y = (i + pad - rr) // stride
                if y >= ho:
                    continue
                for tt in range(s):
                    if (j + pad - tt) % stride or j + pad - tt < 0:
                        continue
                    xo = (j + pad - tt) // stride
                    if xo >= wo:
                        continue
                    dv = F(float(d[nn, kk, y, xo]))
                    dw[kk, cl, rr, tt] += v * dv
                    dz[nn, cc, i, j] += F(float(w[kk, cl, rr, tt])) * dv
    dbias = [sum((F(float(v)) for v in d[:, kk].ravel()), F(0)) for kk in range(k)]
    return dw, dz, dbias


@pytest.mark.parametrize("seed", range(12))
def test_backward_equals_exact_bruteforce_integer(seed):
    x, w, d, stride, pad, groups = _case(seed, integer=True)
    ref = oracle.conv_backward_fp64(x, w, d, stride, pad, groups)
    dw, dz, db = brute_scatter_backward(x, w, d, stride, pad, groups)
    assert np.array_equal(ref["dw"], dw.astype(np.float64))
    assert np.array_equal(ref["dz"], dz.astype(np.float64))
    assert np.array_equal(ref["dbias"], np.array([float(v) for v in db]))


@pytest.mark.parametrize("seed", range(12))
def test_backward_within_rounding_of_exact_bruteforce(seed):
    x, w, d, stride, pad, groups = _case(seed)
    ref = oracle.conv_backward_fp64(x, w, d, stride, pad, groups)
    dw, dz, _ = brute_scatter_backward(x, w, d, stride, pad, groups)
    # fp64 accumulation of m terms: |err| <= m * 2^-53 * mass (m <= 200 here)
    assert np.all(np.abs(ref["dw"] - dw.astype(np.float64)) <= 1e-13 * ref["dw_mass"] + 1e-300)
    assert np.all(np.abs(ref["dz"] - dz.astype(np.float64)) <= 1e-13 * ref["dz_mass"] + 1e-300)


@pytest.mark.parametrize("seed", range(8))
def test_backward_matches_torch_autograd_float64(seed):
    x, w, d, stride, pad, groups = _case(seed + 50)
    xt = torch.from_numpy(x.astype(np.float64)).requires_grad_(True)
    wt = torch.from_numpy(w.astype(np.float64)).requires_grad_(True)
    bt = torch.zeros(w.shape[0], dtype=torch.float64, requires_grad=True)
    out = torch.nn.functional.conv2d(xt, wt, bt, stride=stride, padding=pad, groups=groups)
    out.backward(torch.from_numpy(d.astype(np.float64)))
    ref = oracle.conv_backward_fp64(x, w, d, stride, pad, groups)
    np.testing.assert_allclose(ref["dw"], wt.grad.numpy(), rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(ref["dbias"], bt.grad.numpy(), rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(ref["dz"], xt.grad.numpy() * (x != 0), rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("seed", range(8))
def test_backward_euler_identities(seed):
    """Eq. 1 is linear in W and in `in`: L = <dout, conv(in, W)> = <dw, W> = <dz, in>
    (dz differs from the unmasked gradient only where in == 0)."""
    x, w, d, stride, pad, groups = _case(seed + 100)
    out, _ = oracle.conv_fp64(x, w, None, stride, pad, groups)
    L = float(np.sum(out * d))
    ref = oracle.conv_backward_fp64(x, w, d, stride, pad, groups)
    scale = float(np.sum(np.abs(ref["dw_mass"]) * np.abs(w))) + 1e-300
    assert abs(float(np.sum(ref["dw"] * w)) - L) <= 1e-12 * scale
    assert abs(float(np.sum(ref["dz"] * x)) - L) <= 1e-12 * scale


@pytest.mark.parametrize("groups", [1, 2])
def test_backward_1x1_is_matmul(groups):
    rng = np.random.default_rng(7)
    n, c, h, ww, k = 2, 6, 4, 5, 8
    x = np.where(rng.random((n, c, h, ww)) < 0.5, rng.random((n, c, h, ww)), 0).astype(np.float32)
    w = rng.standard_normal((k, c // groups, 1, 1)).astype(np.float32)
    d = rng.standard_normal((n, k, h, ww)).astype(np.float32)
    ref = oracle.conv_backward_fp64(x, w, d, 1, 0, groups)
    cg, kg = c // groups, k // groups
    for g in range(groups):
        xg = x[:, g * cg:(g + 1) * cg].astype(np.float64).transpose(1, 0, 2, 3).reshape(cg, -1)
        dg = d[:, g * kg:(g + 1) * kg].astype(np.float64).transpose(1, 0, 2, 3).reshape(kg, -1)
        wg = w[g * kg:(g + 1) * kg, :, 0, 0].astype(np.float64)
        np.testing.assert_allclose(ref["dw"][g * kg:(g + 1) * kg, :, 0, 0], dg @ xg.T, rtol=1e-12, atol=1e-12)
        dz = (wg.T @ dg).reshape(cg, n, h, ww).transpose(1, 0, 2, 3) * (x[:, g * cg:(g + 1) * cg] != 0)
        np.testing.assert_allclose(ref["dz"][:, g * cg:(g + 1) * cg], dz, rtol=1e-12, atol=1e-12)


def test_backward_zero_input_and_dbias():
    rng = np.random.default_rng(3)
    x = np.zeros((2, 4, 5, 5), np.float32)
    x[0, 1, 2, 2] = -0.0  # IEEE: -0.0 is zero (R7)
    w = rng.standard_normal((6, 4, 3, 3)).astype(np.float32)
    d = rng.standard_normal((2, 6, 5, 5)).astype(np.float32)
    ref = oracle.conv_backward_fp64(x, w, d, 1, 1, 1)
    assert not ref["dw"].any() and not ref["dz"].any()
    np.testing.assert_allclose(ref["dbias"], d.astype(np.float64).sum(axis=(0, 2, 3)), rtol=1e-13)
