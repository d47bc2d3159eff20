"""Pins for the CPU oracle (oracle/) against things other than itself:
exact-rational brute force in the paper's scatter (ISC) order, torch conv2d in
float64 (a library special case), hand-worked golden fixtures, closed forms and
invariants.  CPU only."""
import fractions
import itertools

import numpy as np
import pytest
import torch

import oracle
from conftest import read_golden_kv
from paper_1704_07724_b200 import datagen


# ---------------------------------------------------------------------------
# independent brute force: ISC scatter order, exact rationals
# ---------------------------------------------------------------------------
def brute_scatter(x, w, b, stride, pad, groups):
    """For every input element (zero or not, so this is the full Eq. 1 sum),
    every output channel k of its group and every tap (r,t): the inverse map
    y = (i+P-r)/T, xo = (j+P-t)/T (R6) decides which output receives
    x*W.  Exact Fraction arithmetic; returns (out, nterms) as object arrays."""
    n, c, h, ww = x.shape
    k, cg, r, s = w.shape
    kg = k // groups
    ho = (h + 2 * pad - r) // stride + 1
    wo = (ww + 2 * pad - s) // stride + 1
    out = np.empty((n, k, ho, wo), dtype=object)
    cnt = np.zeros((n, k, ho, wo), dtype=np.int64)
    for idx in np.ndindex(out.shape):
        out[idx] = fractions.Fraction(0) if b is None else fractions.Fraction(float(b[idx[1]]))
    for nn, cc, i, j in itertools.product(range(n), range(c), range(h), range(ww)):
        v = fractions.Fraction(float(x[nn, cc, i, j]))
        g = cc // cg
        for kk in range(g * kg, (g + 1) * kg):
            for rr in range(r):
                num_y = i + pad - rr
                if num_y < 0 or num_y % stride:
                    continue
                y = num_y // stride
                if y >= ho:
                    continue
                for tt in range(s):
                    num_x = j + pad - tt
                    if num_x < 0 or num_x % stride:
                        continue
                    xo = num_x // stride
                    if xo >= wo:
                        continue
                    out[nn, kk, y, xo] += v * fractions.Fraction(float(w[kk, cc - g * cg, rr, tt]))
                    if x[nn, cc, i, j] != 0:
                        cnt[nn, kk, y, xo] += 1
    return out, cnt


def _tiny_case(seed, integer):
    rng = np.random.default_rng(1000 + seed)
    groups = int(rng.integers(1, 3))
    n = int(rng.integers(1, 3))
    c = groups * int(rng.integers(1, 3))
    k = groups * int(rng.integers(1, 3))
    h, ww = int(rng.integers(1, 5)), int(rng.integers(1, 5))
    stride = int(rng.integers(1, 3))
    pad = int(rng.integers(0, 3))
    r = int(rng.integers(1, min(4, h + 2 * pad) + 1))
    s = int(rng.integers(1, min(4, ww + 2 * pad) + 1))
    mask = rng.random((n, c, h, ww)) < 0.6
    if integer:
        x = np.where(mask, rng.integers(1, 8, (n, c, h, ww)), 0).astype(np.float32)
        w = rng.integers(-8, 9, (k, c // groups, r, s)).astype(np.float32)
        b = rng.integers(-16, 17, k).astype(np.float32)
    else:
        x = np.where(mask, np.abs(rng.standard_normal((n, c, h, ww))), 0).astype(np.float32)
        w = rng.standard_normal((k, c // groups, r, s)).astype(np.float32)
        b = rng.standard_normal(k).astype(np.float32)
    return x, w, b, stride, pad, groups


@pytest.mark.parametrize("seed", range(20))
def test_oracle_equals_exact_bruteforce_integer(seed):
    """S:371 idea: 20 tiny instances (extents <= 4); with integer data every
    partial sum is exact in double, so the oracle must equal the exact sum."""
    x, w, b, stride, pad, groups = _tiny_case(seed, integer=True)
    out, _ = oracle.conv_fp64(x, w, b, stride, pad, groups)
    ref, _ = brute_scatter(x, w, b, stride, pad, groups)
    assert out.shape == ref.shape
    assert np.array_equal(out, ref.astype(np.float64))


@pytest.mark.parametrize("seed", range(20))
def test_oracle_within_rounding_of_exact_bruteforce(seed):
    """Real-valued data: products of two floats are exact in double, so the
    oracle's error is summation rounding only: <= nterms * 2^-53 * (mass+|b|)."""
    x, w, b, stride, pad, groups = _tiny_case(seed, integer=False)
    out, mass = oracle.conv_fp64(x, w, b, stride, pad, groups)
    ref, _ = brute_scatter(x, w, b, stride, pad, groups)
    nterms = (x.shape[1] // groups) * w.shape[2] * w.shape[3] + 1
    bound = nterms * 2.0 ** -53 * (mass + np.abs(b)[None, :, None, None])
    err = np.abs(out - ref.astype(np.float64))
    assert np.all(err <= bound)


def test_hand_worked_example():
    g = read_golden_kv("hand_example_3x3.txt")
    x = np.array(g["input"], dtype=np.float32).reshape(1, 1, 3, 3)
    w = np.array(g["weight"], dtype=np.float32).reshape(1, 1, 3, 3)
    out, mass = oracle.conv_fp64(x, w, None, 1, 1, 1)
    assert np.array_equal(out.reshape(-1), np.array(g["output"], dtype=np.float64))
    assert oracle.exact_nonzero_macs(x, 1, 3, 3, 1, 1) == int(g["exact_macs"][0])
    assert oracle.dense_macs(1, 1, 3, 3, 1, 3, 3, 1, 1) == int(g["dense_macs"][0])
    # ISC step 1: the nonzero values with their row and column, row-major
    lst = oracle.compact_lists(x)
    assert lst["th"] == 3 and lst["tiles"] == 1 and int(lst["counts"][0, 0, 0]) == 2
    assert list(lst["values"][0, 0, 0, :2]) == [int(np.float32(v).view(np.uint32)) for v in g["list_values"]]
    assert list(lst["rows"][0, 0, 0, :2]) == [int(v) for v in g["list_rows"]]
    assert list(lst["cols"][0, 0, 0, :2]) == [int(v) for v in g["list_cols"]]


def _torch_ref(x, w, b, stride, pad, groups):
    return torch.nn.functional.conv2d(
        torch.from_numpy(x).double(), torch.from_numpy(w).double(),
        None if b is None else torch.from_numpy(b).double(),
        stride=stride, padding=pad, groups=groups).numpy()


@pytest.mark.parametrize("seed", range(6))
def test_oracle_matches_torch_conv2d_float64_random(seed):
    rng = np.random.default_rng(seed)
    groups = [1, 2, 4][seed % 3]
    c, k = groups * int(rng.integers(1, 5)), groups * int(rng.integers(1, 5))
    h, ww = int(rng.integers(3, 12)), int(rng.integers(3, 12))
    stride, pad = int(rng.integers(1, 4)), int(rng.integers(0, 3))
    r, s = int(rng.integers(1, 6)), int(rng.integers(1, 6))
    r, s = min(r, h + 2 * pad), min(s, ww + 2 * pad)
    x = (np.abs(rng.standard_normal((2, c, h, ww))) * (rng.random((2, c, h, ww)) > 0.5)).astype(np.float32)
    w = rng.standard_normal((k, c // groups, r, s)).astype(np.float32)
    b = rng.standard_normal(k).astype(np.float32)
    out, mass = oracle.conv_fp64(x, w, b, stride, pad, groups)
    ref = _torch_ref(x, w, b, stride, pad, groups)
    assert out.shape == ref.shape
    np.testing.assert_allclose(out, ref, rtol=0, atol=1e-12)
    # mass is the same contraction applied to |in| and |W| (no bias)
    mref = _torch_ref(np.abs(x), np.abs(w), None, stride, pad, groups)
    np.testing.assert_allclose(mass, mref, rtol=1e-13, atol=1e-300)


def test_oracle_matches_torch_on_table2_shapes(table2):
    """All 10 shapes of Table 2, s in {0, 0.5, 0.9, 0.95}."""
    for i, row in enumerate(table2):
        for sp in (0.0, 0.5, 0.9, 0.95):
            rng = np.random.default_rng(7 * i + int(sp * 100))
            x = (np.abs(rng.standard_normal((1, row["C"], row["H"], row["W"])))
                 * (rng.random((1, row["C"], row["H"], row["W"])) >= sp)).astype(np.float32)
            w = rng.standard_normal((row["K"], row["C"], row["R"], row["S"])).astype(np.float32)
            b = rng.standard_normal(row["K"]).astype(np.float32)
            out, _ = oracle.conv_fp64(x, w, b, row["T"], row["P"], 1)
            ref = _torch_ref(x, w, b, row["T"], row["P"], 1)
            np.testing.assert_allclose(out, ref, rtol=1e-12, atol=1e-11)


# ---------------------------------------------------------------------------
# invariants named by the north star
# ---------------------------------------------------------------------------
def test_zero_input_gives_bias_exactly():
    x = np.zeros((2, 6, 7, 5), np.float32)
    rng = np.random.default_rng(3)
    w = rng.standard_normal((4, 3, 3, 3)).astype(np.float32)
    b = rng.standard_normal(4).astype(np.float32)
    out, mass = oracle.conv_fp64(x, w, b, 2, 1, 2)
    assert np.array_equal(out, np.broadcast_to(b.astype(np.float64)[None, :, None, None], out.shape))
    assert np.all(mass == 0)


def test_linearity_in_input_and_weights():
    """Integer data keeps every sum exact, so linearity holds bit for bit."""
    rng = np.random.default_rng(4)
    x1 = rng.integers(0, 8, (2, 4, 6, 6)).astype(np.float32)
    x2 = rng.integers(0, 8, (2, 4, 6, 6)).astype(np.float32)
    w1 = rng.integers(-8, 9, (6, 2, 3, 3)).astype(np.float32)
    w2 = rng.integers(-8, 9, (6, 2, 3, 3)).astype(np.float32)
    a, bb = 3.0, -2.0
    f = lambda x, w: oracle.conv_fp64(x, w, None, 1, 1, 2)[0]
    assert np.array_equal(f((a * x1 + bb * x2).astype(np.float32), w1), a * f(x1, w1) + bb * f(x2, w1))
    assert np.array_equal(f(x1, (a * w1 + bb * w2).astype(np.float32)), a * f(x1, w1) + bb * f(x1, w2))


@pytest.mark.parametrize("stride,pad", [(1, 1), (1, 0), (2, 1), (1, 2)])
def test_single_nonzero_reproduces_flipped_footprint(stride, pad):
    """One nonzero v at (c,i,j), bias 0: out[k,y,x] = v*W[k,c,i+P-yT,j+P-xT]
    when that tap exists, else 0 (S:251 'kernel spatially flipped')."""
    rng = np.random.default_rng(5)
    c, h, ww, k, r, s = 3, 7, 6, 4, 3, 5
    x = np.zeros((1, c, h, ww), np.float32)
    ci, i, j = 1, 3, 2
    v = np.float32(1.75)
    x[0, ci, i, j] = v
    w = rng.standard_normal((k, c, r, s)).astype(np.float32)
    out, _ = oracle.conv_fp64(x, w, None, stride, pad, 1)
    exp = np.zeros_like(out)
    for kk, y, xo in np.ndindex(k, out.shape[2], out.shape[3]):
        rr, tt = i + pad - y * stride, j + pad - xo * stride
        if 0 <= rr < r and 0 <= tt < s:
            exp[0, kk, y, xo] = np.float64(v) * np.float64(w[kk, ci, rr, tt])
    assert np.array_equal(out, exp)


# ---------------------------------------------------------------------------
# shapes and MAC accounting
# ---------------------------------------------------------------------------
def test_output_shape_floor_form(table2):
    g = read_golden_kv("mac_counts.txt")
    lenet = table2[0]
    shp = oracle.output_shape(1, lenet["C"], lenet["H"], lenet["W"], lenet["K"], lenet["R"], lenet["S"],
                              lenet["T"], lenet["P"])
    assert shp[2:] == (5, 5)
    for row in table2:
        if row["T"] == 1:  # paper's (H+2P-R+1)/T agrees with the floor form at T=1
            ho = oracle.output_shape(1, row["C"], row["H"], row["W"], row["K"], row["R"], row["S"],
                                     row["T"], row["P"])[2]
            assert ho == (row["H"] + 2 * row["P"] - row["R"] + 1) // row["T"]
    with pytest.raises(ValueError):
        oracle.output_shape(1, 1, 2, 2, 1, 5, 5, 1, 0)
    with pytest.raises(ValueError):
        oracle.output_shape(1, 3, 4, 4, 2, 1, 1, 1, 0, groups=2)


def test_mac_counts_golden(table2):
    g = read_golden_kv("mac_counts.txt")
    l = table2[0]
    dm = oracle.dense_macs(1, l["C"], l["H"], l["W"], l["K"], l["R"], l["S"], l["T"], l["P"])
    assert dm == int(g["lenet_conv2_dense"][0])
    assert round(0.05 * dm) == int(g["lenet_conv2_estimated_rho005"][0])
    i5 = table2[7]
    assert oracle.dense_macs(1, i5["C"], i5["H"], i5["W"], i5["K"], 1, 1) == int(g["inception5a2_dense"][0])
    x = np.zeros((1, 1, 7, 7), np.float32)
    x[0, 0, 3, 3] = 1.0
    assert oracle.exact_nonzero_macs(x, 1, 3, 3, 1, 1) == int(g["centre_onehot_exact"][0])
    a4 = table2[2]
    assert a4["R"] * a4["S"] * a4["C"] == int(g["alexneti_conv4_im2col_rows"][0])
    ho = oracle.output_shape(1, a4["C"], a4["H"], a4["W"], a4["K"], 3, 3, 1, 1)[2]
    assert ho * ho == int(g["alexneti_conv4_im2col_cols"][0])


@pytest.mark.parametrize("seed", range(8))
def test_exact_macs_equal_bruteforce_nonzero_terms(seed):
    x, w, b, stride, pad, groups = _tiny_case(seed, integer=True)
    _, cnt = brute_scatter(x, w, b, stride, pad, groups)
    assert oracle.exact_nonzero_macs(x, w.shape[0], w.shape[2], w.shape[3], stride, pad, groups) == cnt.sum()


def test_mac_conservation_at_zero_sparsity(table2):
    """s=0: exact = dense when no tap lands in padding (P=0, T=1);
    with padding, exact = dense - (taps landing in the padding)."""
    for row in table2:
        x = np.ones((1, row["C"], row["H"], row["W"]), np.float32)
        ex = oracle.exact_nonzero_macs(x, row["K"], row["R"], row["S"], row["T"], row["P"])
        dm = oracle.dense_macs(1, row["C"], row["H"], row["W"], row["K"], row["R"], row["S"], row["T"], row["P"])
        if row["P"] == 0 and row["T"] == 1:
            assert ex == dm
        # count in-range taps directly
        _, _, ho, wo = oracle.output_shape(1, row["C"], row["H"], row["W"], row["K"], row["R"], row["S"],
                                           row["T"], row["P"])
        iy = sum(1 for y in range(ho) for r in range(row["R"]) if 0 <= y * row["T"] + r - row["P"] < row["H"])
        ix = sum(1 for xo in range(wo) for t in range(row["S"]) if 0 <= xo * row["T"] + t - row["P"] < row["W"])
        assert ex == row["K"] * row["C"] * iy * ix
        if row["P"] == 0 and row["R"] == 1:
            assert oracle.estimated_macs(x, row["K"], 1, 1) == ex


# ---------------------------------------------------------------------------
# compaction (ISC step 1): per (image, channel, row tile) nonzero values
# with their row and column
# ---------------------------------------------------------------------------
def test_list_rows_rule():
    """whole plane when H*W <= 256, else TH*W <= 256 (>= 1 row)."""
    assert oracle.list_rows(13, 13) == (13, 1, 1)      # 169 elements: one list per plane
    assert oracle.list_rows(12, 12) == (12, 1, 1)
    assert oracle.list_rows(16, 16) == (16, 1, 1)      # exactly 256
    assert oracle.list_rows(28, 28) == (9, 4, 1)       # 9*28 = 252
    assert oracle.list_rows(27, 27) == (9, 3, 1)       # 9*27 = 243
    assert oracle.list_rows(4, 300) == (1, 4, 2)       # one row is wider than 256: u16 index


@pytest.mark.parametrize("shape,th", [((2, 3, 13, 13), None), ((2, 3, 13, 13), 4), ((1, 2, 28, 28), None),
                                      ((2, 2, 27, 27), 1), ((3, 2, 1, 1), None), ((1, 1, 5, 300), None)])
def test_compact_lists_against_numpy_and_roundtrip(shape, th):
    """Each list = np.nonzero of its rows (row-major), values as bit copies; the
    decompressed lists give back the input bit for bit."""
    rng = np.random.default_rng(sum(shape))
    x = (np.abs(rng.standard_normal(shape)) * (rng.random(shape) > 0.85)).astype(np.float32)
    lst = oracle.compact_lists(x, th)
    n, c, h, w = shape
    th = lst["th"]
    assert lst["tiles"] == -(-h // th)
    for ni in range(n):
        for ci in range(c):
            for t in range(lst["tiles"]):
                sub = x[ni, ci, t * th:(t + 1) * th]
                ii, jj = np.nonzero(sub)
                k = int(lst["counts"][ni, ci, t])
                assert k == len(ii) == np.count_nonzero(sub)
                assert np.array_equal(lst["values"][ni, ci, t, :k], sub[ii, jj].view(np.uint32))
                assert np.array_equal(lst["rows"][ni, ci, t, :k], ii + t * th)
                assert np.array_equal(lst["cols"][ni, ci, t, :k], jj)
    back = oracle.decompress_lists(lst, shape)
    assert np.array_equal(back.view(np.uint32), x.view(np.uint32))


def test_compact_lists_zero_semantics():
    """R7: IEEE compare x != 0.0f: -0.0 is zero; subnormals, NaN, Inf are not."""
    x = np.zeros((1, 1, 2, 4), np.float32)
    x[0, 0, 0, 0] = -0.0
    x[0, 0, 0, 1] = np.float32(1e-45)          # smallest subnormal
    x[0, 0, 0, 2] = np.nan
    x[0, 0, 1, 0] = np.inf
    x[0, 0, 1, 3] = -2.5
    lst = oracle.compact_lists(x)
    assert int(lst["counts"][0, 0, 0]) == 4
    assert list(lst["rows"][0, 0, 0, :4]) == [0, 0, 1, 1]
    assert list(lst["cols"][0, 0, 0, :4]) == [1, 2, 0, 3]
    assert lst["values"][0, 0, 0, 0] == np.float32(1e-45).view(np.uint32)
    assert lst["values"][0, 0, 0, 3] == np.float32(-2.5).view(np.uint32)


def test_sparsity_pins():
    """sparsity = 1 - #nonzeros/size, exact IEEE zero test (R7).
    7 nonzeros (a subnormal, NaN, Inf and negative values among them) in 100
    elements with a -0.0 -> 0.93; all-zero -> 1; dense -> 0."""
    x = np.zeros(100, np.float32)
    x[3] = -0.0
    x[[5, 17, 40]] = [1.0, -3.0, 0.5]
    x[50] = np.float32(1e-45)
    x[60] = np.nan
    x[70] = -np.inf
    x[99] = 2.0
    assert oracle.sparsity(x) == pytest.approx(0.93, abs=1e-15)
    assert oracle.sparsity(np.zeros((4, 5), np.float32)) == 1.0
    assert oracle.sparsity(np.ones((3, 3), np.float32)) == 0.0
    assert oracle.sparsity(-np.zeros(8, np.float32)) == 1.0


# ---------------------------------------------------------------------------
# generators
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("s", [0.9, 0.95, 0.99])
def test_generator_sparsity_within_binomial_ci(s):
    shp = datagen.C2.with_batch(4)
    x = datagen.activations(shp, s)
    n = x.size
    nz = np.count_nonzero(x)
    p = 1 - s
    sd = np.sqrt(n * p * (1 - p))
    assert abs(nz - n * p) <= 3.3 * sd   # 99.9% two-sided
    assert np.all(x >= 0)


def test_generator_counter_based_slices():
    shp = datagen.C4B.with_batch(8)
    full = datagen.activations(shp, 0.95)
    part = datagen.activations(shp, 0.95, start=5, count=3)
    assert np.array_equal(full[5:8], part)


def test_generator_c3_dead_channels():
    shp = datagen.C3.with_batch(3)
    s_c = datagen.channel_sparsity(shp)
    assert int(np.sum(s_c == 1.0)) == 5
    x = datagen.activations(shp, "channel")
    dead = np.where(s_c == 1.0)[0]
    assert np.all(x[:, dead] == 0)
    live = s_c < 1
    assert np.all((s_c[live] >= 0.85) & (s_c[live] < 0.99))


def test_relu_of_symmetric_tensor_half_sparse():
    """relu of a zero-mean symmetric 1e6-element tensor -> s = 0.5 +- 0.02."""
    rng = np.random.default_rng(11)
    t = rng.standard_normal(10 ** 6).astype(np.float32)
    z = oracle.relu(t)
    assert abs(oracle.sparsity(z) - 0.5) <= 0.02
    assert np.array_equal(oracle.relu(z), z)
    assert np.all(z >= 0)
