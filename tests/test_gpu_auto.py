"""GPU tests of the device-side sparse <-> dense crossover (
the paper's regime "speedup ... when the sparsity is not less than 0.9",
PAPER.md:23): sparse_conv_forward_auto counts the batch's nonzeros on
the device and gates the two enqueued paths.

Checks: the nonzero count equals the input's (exact integer), the path taken
is the one the rule s >= s* prescribes, the output meets the bar of the path
taken (sparse: 1e-5 * mass + 1e-6; dense: TF32 2^-9 * mass + 1e-6; both
against the oracle), the decision follows the data under CUDA-graph replay
(no host round trip), and calibration returns a crossover consistent with
the times it measured."""
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


def make_conv(sc, shp, w, b, max_batch=None):
    return sc.SparseConv(torch.from_numpy(w).to(DEV), None if b is None else torch.from_numpy(b).to(DEV),
                         max_batch or shp.n, shp.c, shp.h, shp.w, shp.stride, shp.pad, shp.groups)


def check(got, x, w, b, shp, path, sc):
    for i0 in range(x.shape[0]):
        ref, mass = oracle.conv_fp64(x[i0:i0 + 1], w, b, shp.stride, shp.pad, shp.groups)
        tol = oracle.tolerance_sparse(mass) if path == sc.SC_PATH_SPARSE else oracle.tolerance_dense_tf32(mass)
        err = np.abs(got[i0:i0 + 1].astype(np.float64) - ref)
        assert np.all(err <= tol), f"image {i0} path {path}: max err/tol {(err / tol).max():.3f}"


def expected_path(sc, x, s_star):
    nnz = int(np.count_nonzero(x))
    return (sc.SC_PATH_SPARSE if nnz <= (1.0 - s_star) * x.size else sc.SC_PATH_DENSE), nnz


@pytest.mark.parametrize("cfg", ["C2", "C4b"])
@pytest.mark.parametrize("s", [0.0, 0.5, 0.9, 0.95, 0.99])
def test_auto_rule_and_parity(sc, cfg, s):
    shp = datagen.CONFIGS[cfg].with_batch(3)
    x = datagen.activations(shp, s, seed=11)
    w, b = datagen.weights(shp, seed=11)
    conv = make_conv(sc, shp, w, b, max_batch=4)
    conv.crossover = 0.9  # the paper's regime
    out = conv.forward_auto(torch.from_numpy(x).to(DEV)).cpu().numpy()
    path, nnz = conv.last_path()
    want, nnz_ref = expected_path(sc, x, 0.9)
    assert nnz == nnz_ref
    assert path == want
    check(out, x, w, b, shp, path, sc)


def test_auto_extreme_thresholds(sc):
    shp = datagen.C2.with_batch(2)
    x = datagen.activations(shp, 0.5, seed=3)
    w, b = datagen.weights(shp, seed=3)
    conv = make_conv(sc, shp, w, b)
    xd = torch.from_numpy(x).to(DEV)
    conv.crossover = 0.0  # s >= 0 always: sparse
    out = conv.forward_auto(xd).cpu().numpy()
    assert conv.last_path()[0] == sc.SC_PATH_SPARSE
    check(out, x, w, b, shp, sc.SC_PATH_SPARSE, sc)
    conv.crossover = 1.0  # only an all-zero batch is sparse enough
    out = conv.forward_auto(xd).cpu().numpy()
    assert conv.last_path()[0] == sc.SC_PATH_DENSE
    check(out, x, w, b, shp, sc.SC_PATH_DENSE, sc)
    z = np.zeros_like(x)
    out = conv.forward_auto(torch.from_numpy(z).to(DEV)).cpu().numpy()
    assert conv.last_path() == (sc.SC_PATH_SPARSE, 0)
    assert np.array_equal(out, np.broadcast_to(b[None, :, None, None], out.shape))
    with pytest.raises(sc.SparseConvError):
        conv.crossover = 1.5


def test_auto_exact_boundary(sc):
    """nnz == (1 - s*) * elems exactly is sparse (s >= s*); one more nonzero is dense."""
    shp = datagen.C4B.with_batch(1)
    elems = shp.c * shp.h * shp.w  # 12544
    w, b = datagen.weights(shp, seed=5)
    conv = make_conv(sc, shp, w, b)
    conv.crossover = 0.75  # limit = 3136 nonzeros, exact in binary
    rng = np.random.default_rng(5)
    for nnz, want in ((3136, sc.SC_PATH_SPARSE), (3137, sc.SC_PATH_DENSE)):
        x = np.zeros(elems, np.float32)
        x[rng.choice(elems, nnz, replace=False)] = rng.random(nnz, dtype=np.float32) + 0.5
        x = x.reshape(1, shp.c, shp.h, shp.w)
        out = conv.forward_auto(torch.from_numpy(x).to(DEV)).cpu().numpy()
        assert conv.last_path() == (want, nnz)
        check(out, x, w, b, shp, want, sc)


def test_auto_graph_replay_follows_data(sc):
    """The decision is taken on the device at replay time."""
    shp = datagen.C2.with_batch(4)
    w, b = datagen.weights(shp, seed=9)
    conv = make_conv(sc, shp, w, b)
    conv.crossover = 0.9
    xs = {s: datagen.activations(shp, s, seed=9) for s in (0.5, 0.99)}
    xin = torch.from_numpy(xs[0.5]).to(DEV)
    out = torch.empty((shp.n, shp.k, shp.ho, shp.wo), device=DEV)
    stream = torch.cuda.Stream()
    with torch.cuda.stream(stream):
        conv.forward_auto(xin, out, stream=stream)  # warm-up outside capture
        stream.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=stream):
            conv.forward_auto(xin, out, stream=stream)
    for s in (0.99, 0.5, 0.99):
        xin.copy_(torch.from_numpy(xs[s]))
        out.fill_(float("nan"))
        g.replay()
        torch.cuda.synchronize()
        path, nnz = conv.last_path()
        assert nnz == int(np.count_nonzero(xs[s]))
        assert path == (sc.SC_PATH_SPARSE if s == 0.99 else sc.SC_PATH_DENSE)
        check(out.cpu().numpy(), xs[s], w, b, shp, path, sc)


def test_auto_dense_unsupported_is_sparse(sc):
    """W_out > 256 has no dense path: always sparse, calibration says s* = 0."""
    shp = datagen.ConvShape("wide", 99, 2, 4, 3, 300, 8, 3, 3, 1, 1, 1)
    x = datagen.activations(shp, 0.0, seed=1)
    w, b = datagen.weights(shp, seed=1)
    conv = make_conv(sc, shp, w, b)
    assert conv.calibrate_crossover(2) == 0.0
    out = conv.forward_auto(torch.from_numpy(x).to(DEV)).cpu().numpy()
    assert conv.last_path() == (sc.SC_PATH_SPARSE, int(np.count_nonzero(x)))
    check(out, x, w, b, shp, sc.SC_PATH_SPARSE, sc)


@pytest.mark.parametrize("cfg", ["C2", "C4b"])
def test_auto_calibration(sc, cfg):
    """Calibrated s* in [0, 1]; an uncalibrated plan calibrates on first use;
    timing the two paths on batches on either side of s* agrees with it
    (with a margin for timing noise)."""
    shp = datagen.CONFIGS[cfg]
    w, b = datagen.weights(shp, seed=2)
    conv = make_conv(sc, shp, w, b)
    assert conv.crossover is None
    x = datagen.activations(shp, 0.95, seed=2, count=8)
    xin = torch.from_numpy(np.ascontiguousarray(x)).to(DEV)
    conv.forward_auto(xin)  # calibrates for n = 8
    s8 = conv.crossover
    assert s8 is not None and 0.0 <= s8 <= 1.0
    s_star = conv.calibrate_crossover(shp.n)
    assert 0.0 <= s_star <= 1.0
    full = torch.from_numpy(datagen.activations(shp, 0.5, seed=2)).to(DEV)
    out = torch.empty((shp.n, shp.k, shp.ho, shp.wo), device=DEV)

    def t(fn):
        for _ in range(2):
            fn(full, out)
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        ev[0].record()
        for _ in range(5):
            fn(full, out)
        ev[1].record()
        torch.cuda.synchronize()
        return ev[0].elapsed_time(ev[1]) / 5

    if s_star < 0.45:  # sparse must then not lose badly at s = 0.5
        assert t(conv.forward) <= 1.3 * t(conv.dense_forward)
    elif s_star > 0.55:
        assert t(conv.dense_forward) <= 1.3 * t(conv.forward)
    conv.forward_auto(full, out)
    path, _ = conv.last_path()
    assert path == expected_path(sc, full.cpu().numpy(), s_star)[0]


def test_auto_launch_count(sc):
    shp = datagen.C2.with_batch(2)
    w, b = datagen.weights(shp)
    conv = make_conv(sc, shp, w, b)
    sp, de = conv.launch_counts
    assert (sp, de) == (3, 2)
