"""sparse_conv_forward_batches: independent batches pipelined across two stage-1 workspaces and
prioritized streams.  The same kernels run as in
sparse_conv_forward, so every batch's output must be bit-identical to a plain forward of that
batch; sampled images are also checked against the oracle (1e-5 * mass)."""
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


def make(sc, shp, seed=0, max_batch=None):
    w, b = datagen.weights(shp, seed=seed)
    conv = sc.SparseConv(torch.from_numpy(w).to(DEV), torch.from_numpy(b).to(DEV), max_batch or shp.n, shp.c, shp.h,
                         shp.w, shp.stride, shp.pad, shp.groups)
    return conv, w, b


def batches(shp, s, nbatch, n):
    return [torch.from_numpy(datagen.activations(shp.with_batch(n), s, seed=100 + i)).to(DEV) for i in range(nbatch)]


def check_oracle(out, x, w, b, shp, images):
    for i in images:
        ref, mass = oracle.conv_fp64(x[i:i + 1].cpu().numpy(), w, b, shp.stride, shp.pad, shp.groups)
        assert np.all(np.abs(out[i:i + 1].cpu().numpy() - ref) <= oracle.tolerance_sparse(mass))


CASES = [("C2", 0.95, 5, 6), ("C2", 0.9, 3, 128), ("C4a", 0.95, 4, 5), ("C4b", 0.99, 4, 7), ("C1", 0.9, 3, 9),
         ("C3", "channel", 3, 4)]


@pytest.mark.parametrize("cfg,s,nbatch,n", CASES)
def test_batches_bitexact_vs_forward(sc, cfg, s, nbatch, n):
    """Every batch bit-identical to sparse_conv_forward of that batch (n = 128: the bench's
    launch configuration), first and last images of every batch against the oracle."""
    shp = datagen.CONFIGS[cfg]
    conv, w, b = make(sc, shp)
    xs = batches(shp, s, nbatch, n)
    outs = conv.forward_batches(xs)
    torch.cuda.synchronize()
    for x, o in zip(xs, outs):
        assert torch.equal(o, conv.forward(x))
        check_oracle(o, x, w, b, shp, [0, n - 1])


def test_batches_other_kernels(sc, monkeypatch):
    """A Table 2 variant, a run-time generated tiling and the generic kernel behind the pipeline."""
    t2 = {t.name: t for t, _ in datagen.table2_shapes(n=3)}
    shapes = [(t2["GoogLeNet-Inception5a.1"], None), (datagen.ConvShape("batches_jit", 991, 3, 12, 20, 20, 130, 3, 3, 1,
                                                                         1, 1), None),
              (datagen.CONFIGS["C2"].with_batch(3), "0")]
    for shp, force in shapes:
        if force is None:
            monkeypatch.delenv("SC_FORCE_VARIANT", raising=False)
        else:
            monkeypatch.setenv("SC_FORCE_VARIANT", force)
        conv, w, b = make(sc, shp)
        xs = batches(shp, 0.9, 4, 3)
        outs = conv.forward_batches(xs)
        torch.cuda.synchronize()
        for x, o in zip(xs, outs):
            assert torch.equal(o, conv.forward(x)), (shp.name, conv.variant)
            check_oracle(o, x, w, b, shp, [0, 2])


def test_batches_single_and_interleaved(sc):
    """nbatch = 1 is sparse_conv_forward; plain forwards before and after a batches call (the
    plan's own workspace is slot 0 of the pipeline) stay correct."""
    shp = datagen.CONFIGS["C2"].with_batch(4)
    conv, w, b = make(sc, shp)
    xs = batches(shp, 0.95, 5, 4)
    ref = [conv.forward(x).clone() for x in xs]
    assert torch.equal(conv.forward_batches(xs[:1])[0], ref[0])
    y0 = conv.forward(xs[0])
    outs = conv.forward_batches(xs)
    y1 = conv.forward(xs[1])
    torch.cuda.synchronize()
    assert torch.equal(y0, ref[0]) and torch.equal(y1, ref[1])
    for o, r in zip(outs, ref):
        assert torch.equal(o, r)


def test_batches_ragged_n(sc):
    shp = datagen.CONFIGS["C4b"]
    conv, w, b = make(sc, shp.with_batch(8))
    xs = batches(shp, 0.95, 3, 5)  # n = 5 of an 8-image plan
    outs = conv.forward_batches(xs)
    torch.cuda.synchronize()
    for x, o in zip(xs, outs):
        assert torch.equal(o, conv.forward(x))


def test_batches_graph_capture(sc):
    """Capture after sparse_conv_reserve_batches; replays match; the first call under capture
    without the reservation is refused."""
    shp = datagen.CONFIGS["C2"].with_batch(4)
    conv, w, b = make(sc, shp)
    xs = batches(shp, 0.95, 4, 4)
    ref = [conv.forward(x).clone() for x in xs]
    outs = [torch.empty_like(r) for r in ref]
    fresh, _, _ = make(sc, shp)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        g = torch.cuda.CUDAGraph()
        with pytest.raises(sc.SparseConvError) as e:
            with torch.cuda.graph(g, stream=s):
                fresh.forward_batches(xs, outs, stream=s)
        assert e.value.status == 1 and "reserve" in str(e.value)
    torch.cuda.synchronize()
    conv.reserve_batches()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        conv.forward_batches(xs, outs, stream=s)
    for _ in range(3):
        for o in outs:
            o.zero_()
        g.replay()
        torch.cuda.synchronize()
        for o, r in zip(outs, ref):
            assert torch.equal(o, r)


def test_batches_bad_arguments(sc):
    shp = datagen.CONFIGS["C4b"].with_batch(2)
    conv, _, _ = make(sc, shp)
    x = batches(shp, 0.9, 1, 2)[0]
    import ctypes
    with pytest.raises(sc.SparseConvError) as e:
        sc._check(sc.lib().sparse_conv_forward_batches(conv._plan, 0, 2, None, None, None))
    assert e.value.status == 1
    ins = (ctypes.c_void_p * 2)(x.data_ptr(), 0)
    ous = (ctypes.c_void_p * 2)(x.data_ptr(), x.data_ptr())
    with pytest.raises(sc.SparseConvError) as e:
        sc._check(sc.lib().sparse_conv_forward_batches(conv._plan, 2, 2, ins, ous, None))
    assert e.value.status == 1


@pytest.mark.parametrize("cfg,n,nbatch", [("C2", 128, 5), ("C4b", 7, 4), ("C1", 9, 3), ("C2", 6, 1)])
def test_host_batches_match_device_forward(sc, cfg, n, nbatch):
    """sparse_conv_forward_host_batches: pinned host batches through the chunked copy/compute
    pipeline continued across batches (two staging sets); every batch's host output equals the
    device forward of that batch bit for bit (same kernels), the first and last images of the
    first and last batches against the oracle."""
    shp = datagen.CONFIGS[cfg]
    conv, w, b = make(sc, shp, max_batch=max(n, 8))
    xs = [torch.from_numpy(datagen.activations(shp.with_batch(n), 0.9, seed=200 + i)) for i in range(nbatch)]
    h_in = [x.pin_memory() for x in xs]
    h_out = [torch.empty((n,) + conv.out_shape).pin_memory() for _ in range(nbatch)]
    conv.forward_host_batches(h_in, h_out)
    for i, (x, o) in enumerate(zip(xs, h_out)):
        assert torch.equal(o, conv.forward(x.to(DEV)).cpu()), f"batch {i}"
    for i in sorted({0, nbatch - 1}):
        check_oracle(h_out[i], xs[i], w, b, shp, [0, n - 1])


def test_host_batches_bad_arguments(sc):
    import ctypes
    shp = datagen.CONFIGS["C4b"].with_batch(2)
    conv, _, _ = make(sc, shp)
    with pytest.raises(sc.SparseConvError) as e:
        sc._check(sc.lib().sparse_conv_forward_host_batches(conv._plan, 0, 2, None, None, None))
    assert e.value.status == 1
    h = torch.zeros((2,) + conv.in_shape)
    ins = (ctypes.c_void_p * 2)(h.data_ptr(), 0)
    ous = (ctypes.c_void_p * 2)(h.data_ptr(), h.data_ptr())
    with pytest.raises(sc.SparseConvError) as e:
        sc._check(sc.lib().sparse_conv_forward_host_batches(conv._plan, 2, 2, ins, ous, None))
    assert e.value.status == 1
