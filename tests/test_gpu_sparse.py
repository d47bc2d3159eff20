"""GPU parity of the sparse path (C-ABI library) against the CPU oracle.

Bars (north star):
* stage-1 lists bit-exact (counts, values bits, indices; slack never compared);
* outputs within |gpu - oracle| <= 1e-5 * mass + 1e-6 per element;
* integer-valued data: bit-exact (every partial sum is exact in fp32).
Full BASELINE sizes run in the bench's launch configuration (same plan, full
batch); the oracle then checks sampled images (images are independent,
Eq. 1 has no cross-image term)."""
import numpy as np
import pytest
import torch

import oracle
from paper_1704_07724_b200 import datagen
from lists_check import check_plane_lists, check_streams

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


# Tile height the stage-2 stream layout uses for each BASELINE config (the shipped
# variants): stated here so a plan that silently changed its
# layout fails the stream check instead of being compared against itself.
EXPECTED_TY = {"C1": 1, "C2": 2, "C3": 3, "C4a": 2, "C4b": 3}


def check_lists(conv, x, n, cfg=None):
    """Stage 1 bit-exact: (a) the paper-level lists against
    oracle.compact_lists; (b) the stage-2 streams against the test-side
    adapter's derivation from the same oracle lists (tests/r9_adapter.py)."""
    check_plane_lists(conv, x, n)
    check_streams(conv, x, n, EXPECTED_TY.get(cfg))


def check_conv(got, x, w, b, shp, relu=False, images=None):
    images = range(x.shape[0]) if images is None else images
    worst = 0.0
    for i0 in images:
        ref, mass = oracle.conv_fp64(x[i0:i0 + 1], w, b, shp.stride, shp.pad, shp.groups)
        if relu:
            ref = np.maximum(ref, 0.0)
        g = got[i0:i0 + 1].astype(np.float64)
        err = np.abs(g - ref)
        tol = oracle.tolerance_sparse(mass)
        bad = err > tol
        assert not bad.any(), (f"image {i0}: {bad.sum()} outputs out of tolerance; "
                               f"max err {err.max():.3e} max ratio {(err / tol).max():.3f}")
        worst = max(worst, float((err / tol).max()))
    return worst


SPARSE_CASES = [("C1", 0.9), ("C2", 0.9), ("C2", 0.95), ("C2", 0.99), ("C3", "channel"), ("C4a", 0.9),
                ("C4a", 0.95), ("C4a", 0.99), ("C4b", 0.9), ("C4b", 0.95), ("C4b", 0.99)]


@pytest.mark.parametrize("cfg,s", SPARSE_CASES)
def test_full_config_lists_bitexact_and_sampled_outputs(sc, cfg, s):
    """BASELINE sizes in the bench's launch configuration: whole batch through
    sparse_conv_forward; lists bit-exact for the whole batch, outputs checked
    on images {0, 1, middle, last}."""
    shp = datagen.CONFIGS[cfg]
    x = datagen.activations(shp, s)
    w, b = datagen.weights(shp)
    conv = make_conv(sc, shp, w, b)
    xd = torch.from_numpy(x).to(DEV)
    out = conv.forward(xd)
    torch.cuda.synchronize()
    check_lists(conv, x, shp.n, cfg)
    got = out.cpu().numpy()
    check_conv(got, x, w, b, shp, images=[0, 1, shp.n // 2, shp.n - 1])


@pytest.mark.parametrize("cfg", ["C1", "C2", "C3", "C4a", "C4b"])
@pytest.mark.parametrize("s", [0.0, 0.5, 0.95])
def test_small_batch_all_outputs(sc, cfg, s):
    """Every output of a 3-image batch (spans all tiles and ragged tails),
    including dense (s=0) input: the sparse path must still meet 1e-5."""
    shp = datagen.CONFIGS[cfg].with_batch(3)
    x = datagen.activations(shp, s if cfg != "C3" or s == 0.0 else "channel", seed=5)
    w, b = datagen.weights(shp, seed=5)
    conv = make_conv(sc, shp, w, b, max_batch=8)
    out = conv.forward(torch.from_numpy(x).to(DEV))
    torch.cuda.synchronize()
    check_lists(conv, x, 3, cfg)
    check_conv(out.cpu().numpy(), x, w, b, shp)


def test_table2_shapes(sc):
    """Paper Table 2 shapes incl. stride 2 and 1x1, at their
    printed sparsity, N=2, all outputs."""
    for shp, s in datagen.table2_shapes(n=2):
        x = datagen.activations(shp, s)
        w, b = datagen.weights(shp)
        conv = make_conv(sc, shp, w, b)
        out = conv.forward(torch.from_numpy(x).to(DEV))
        torch.cuda.synchronize()
        check_lists(conv, x, 2)
        check_conv(out.cpu().numpy(), x, w, b, shp)


@pytest.mark.parametrize("cfg", ["C1", "C2", "C3", "C4a", "C4b"])
def test_integer_data_bitexact(sc, cfg):
    shp = datagen.CONFIGS[cfg].with_batch(4)
    x, w, b = datagen.integer_case(shp, sparsity=0.6)
    conv = make_conv(sc, shp, w, b)
    out = conv.forward(torch.from_numpy(x).to(DEV)).cpu().numpy()
    ref, _ = oracle.conv_fp64(x, w, b, shp.stride, shp.pad, shp.groups)
    assert np.array_equal(out.astype(np.float64), ref)


def test_integer_data_bitexact_table2(sc):
    for shp, _ in datagen.table2_shapes(n=2):
        x, w, b = datagen.integer_case(shp, sparsity=0.7)
        conv = make_conv(sc, shp, w, b)
        out = conv.forward(torch.from_numpy(x).to(DEV)).cpu().numpy()
        ref, _ = oracle.conv_fp64(x, w, b, shp.stride, shp.pad, shp.groups)
        assert np.array_equal(out.astype(np.float64), ref), shp.name


# Stage-2 kernel a plan picks for the 1x1 Table 2 layers (tools/gen_gather.py VARIANTS: the
# wide k-block tilings V53-V56 for Kg >= 150, else the round-1 V43/V45).
T2_1X1_VARIANT = {"GoogLeNet-Inception4a.1": 53, "GoogLeNet-Inception4a.2": 43, "GoogLeNet-Inception5a.1": 54,
                  "GoogLeNet-Inception5a.2": 55}


def test_table2_1x1_variant_choice(sc):
    for shp, _ in datagen.table2_shapes(n=2):
        if shp.name in T2_1X1_VARIANT:
            w, b = datagen.weights(shp)
            assert make_conv(sc, shp, w, b).variant[0] == T2_1X1_VARIANT[shp.name], shp.name


# (Kg, plane width, groups, variant): KL = the fewest k-blocks of 128 / 192 / 256 filters
# (sc_internal.h wide_1x1_kl), Kg >= 150
WIDE_CASES = [(151, 14, 1, 53), (149, 14, 1, 43), (256, 14, 1, 56), (300, 14, 1, 53), (400, 14, 1, 56),
              (201, 7, 1, 54), (199, 7, 1, 54), (150, 7, 1, 55), (192, 7, 1, 55), (149, 7, 1, 45), (300, 7, 1, 55),
              (201, 7, 2, 54)]


@pytest.mark.parametrize("k,wd,groups,want", WIDE_CASES)
def test_wide_kblock_1x1_ragged(sc, k, wd, groups, want):
    """KL = 6 / 8 tiles (k-blocks of 192 / 256 channels) at the rule's edges and with ragged
    last k-blocks (zero-padded weights, pack.cu) and groups: tolerance at s=0.9 on all
    outputs, stage-1 lists bit-exact, integer data bit-exact."""
    shp = datagen.ConvShape(f"wide_kblock_{k}_{wd}_{groups}", 5000 + k + wd, 3, 38 * groups, wd, wd, k * groups, 1, 1,
                            1, 0, groups)
    x = datagen.activations(shp, 0.9, seed=k)
    w, b = datagen.weights(shp, seed=k)
    conv = make_conv(sc, shp, w, b, max_batch=4)
    assert conv.variant[0] == want
    out = conv.forward(torch.from_numpy(x).to(DEV)).cpu().numpy()
    check_lists(conv, x, 3)
    check_conv(out, x, w, b, shp)
    xi, wi, bi = datagen.integer_case(shp, sparsity=0.7)
    conv = make_conv(sc, shp, wi, bi, max_batch=4)
    out = conv.forward(torch.from_numpy(xi).to(DEV)).cpu().numpy()
    ref, _ = oracle.conv_fp64(xi, wi, bi, shp.stride, shp.pad, shp.groups)
    assert np.array_equal(out.astype(np.float64), ref)


@pytest.mark.parametrize("layer,variant", [("GoogLeNet-Inception4a.1", 48), ("GoogLeNet-Inception5a.1", 49)])
def test_superseded_t2_tilings(sc, layer, variant, monkeypatch):
    """The round-1 1x1 tilings V48 / V49 (no longer built in), generated at run time."""
    want = force_kernel(monkeypatch, variant)
    shp = {t.name: t for t, _ in datagen.table2_shapes(n=2)}[layer]
    x = datagen.activations(shp, 0.9, seed=5)
    w, b = datagen.weights(shp, seed=5)
    conv = make_conv(sc, shp, w, b)
    assert conv.variant[0] == want
    out = conv.forward(torch.from_numpy(x).to(DEV)).cpu().numpy()
    check_conv(out, x, w, b, shp)


@pytest.mark.parametrize("cfg", ["C2", "C3", "C4b"])
def test_zero_input_gives_bias(sc, cfg):
    shp = datagen.CONFIGS[cfg].with_batch(2)
    w, b = datagen.weights(shp)
    conv = make_conv(sc, shp, w, b)
    x = torch.zeros((2, shp.c, shp.h, shp.w), device=DEV)
    out = conv.forward(x).cpu().numpy()
    assert np.array_equal(out, np.broadcast_to(b[None, :, None, None], out.shape))
    lists = conv.lists(2)
    assert int(lists["offs"][:, :, -1].sum()) == 0   # R9: no entries, no markers: every stream is empty


@pytest.mark.parametrize("cfg", ["C1", "C2", "C3", "C4a"])
def test_one_hot_flipped_footprint(sc, cfg):
    """Single nonzero v at (c,i,j), bias 0: out = fl32(v*W[k,c,i+P-y,j+P-x]),
    bit-exact (one rounded product per output)."""
    shp = datagen.CONFIGS[cfg].with_batch(1)
    w, _ = datagen.weights(shp)
    conv = make_conv(sc, shp, w, None)
    for (ci, i, j) in [(0, 0, 0), (shp.c - 1, shp.h - 1, shp.w - 1), (shp.c // 2, shp.h // 2, 1)]:
        x = np.zeros((1, shp.c, shp.h, shp.w), np.float32)
        v = np.float32(1.3125)
        x[0, ci, i, j] = v
        out = conv.forward(torch.from_numpy(x).to(DEV)).cpu().numpy()
        g = ci // (shp.c // shp.groups)
        kg = shp.k // shp.groups
        exp = np.zeros_like(out)
        for y in range(shp.ho):
            for xo in range(shp.wo):
                r, t = i + shp.pad - y, j + shp.pad - xo
                if 0 <= r < shp.r and 0 <= t < shp.s:
                    exp[0, g * kg:(g + 1) * kg, y, xo] = v * w[g * kg:(g + 1) * kg, ci % (shp.c // shp.groups), r, t]
        assert np.array_equal(out, exp)


def test_subnormal_inputs_count_as_nonzero(sc):
    """R7: subnormal inputs are nonzero (no FTZ anywhere)."""
    shp = datagen.C2.with_batch(1)
    w, b = datagen.weights(shp)
    conv = make_conv(sc, shp, w, None)
    x = np.zeros((1, shp.c, shp.h, shp.w), np.float32)
    x[0, 3, 5, 6] = np.float32(1e-40)
    x[0, 7, 0, 0] = np.float32(-0.0)
    conv.compact(torch.from_numpy(x).to(DEV))
    torch.cuda.synchronize()
    check_lists(conv, x, 1)
    st = conv.lists(1)
    # R9: in every tile window that holds input row 5, one marker (channel 3) + the subnormal;
    # -0.0 is zero, so channel 7 has no entry and no marker anywhere
    lo = np.arange(st["tiles"]) * st["ty"] * shp.stride - shp.pad
    in_windows = int(((lo <= 5) & (5 < lo + st["nwr"])).sum())
    assert in_windows >= 1
    assert int(st["offs"][0, :, -1].sum()) == 2 * in_windows
    ws = np.full_like(w, 2.0 ** 100)
    conv2 = make_conv(sc, shp, ws, None)
    out = conv2.forward(torch.from_numpy(x).to(DEV)).cpu().numpy()
    assert out[0, 0, 5, 6] == np.float32(np.float64(np.float32(1e-40)) * 2.0 ** 100)


def test_ragged_batch_and_determinism(sc):
    shp = datagen.C2.with_batch(5)
    x = datagen.activations(shp, 0.95)
    w, b = datagen.weights(shp)
    conv = make_conv(sc, shp, w, b, max_batch=16)
    xd = torch.from_numpy(x).to(DEV)
    o1 = conv.forward(xd).cpu().numpy()
    o2 = conv.forward(xd).cpu().numpy()
    assert np.array_equal(o1.view(np.uint32), o2.view(np.uint32))
    o3 = conv.forward(xd[:2].contiguous()).cpu().numpy()
    assert np.array_equal(o3.view(np.uint32), o1[:2].view(np.uint32))
    check_conv(o1, x, w, b, shp)


def test_fused_relu_flag(sc):
    shp = datagen.C2.with_batch(2)
    x = datagen.activations(shp, 0.9)
    w, b = datagen.weights(shp)
    conv = make_conv(sc, shp, w, b, relu=True)
    out = conv.forward(torch.from_numpy(x).to(DEV)).cpu().numpy()
    assert out.min() >= 0.0
    check_conv(out, x, w, b, shp, relu=True)


def test_forward_host_matches_device(sc):
    shp = datagen.C4B.with_batch(6)
    x = datagen.activations(shp, 0.95)
    w, b = datagen.weights(shp)
    conv = make_conv(sc, shp, w, b)
    dev = conv.forward(torch.from_numpy(x).to(DEV)).cpu()
    h_in = torch.from_numpy(x).pin_memory()
    h_out = torch.empty((6,) + conv.out_shape).pin_memory()
    conv.forward_host(h_in, h_out)
    assert torch.equal(dev, h_out)


@pytest.mark.parametrize("n,pinned", [(37, True), (16, False), (128, True)])
def test_forward_host_pipelined_chunks(sc, n, pinned):
    """The host path cuts the batch into up to 4 chunks (boundaries at multiples of
    4 images, ragged last chunk) on its own streams: identical to the device path."""
    shp = datagen.C2.with_batch(n)
    x = datagen.activations(shp, 0.95, seed=17)
    w, b = datagen.weights(shp, seed=17)
    conv = make_conv(sc, shp, w, b, max_batch=128)
    dev = conv.forward(torch.from_numpy(x).to(DEV)).cpu()
    h_in = torch.from_numpy(x)
    h_out = torch.full((n,) + conv.out_shape, float("nan"))
    if pinned:
        h_in, h_out = h_in.pin_memory(), h_out.pin_memory()
    conv.forward_host(h_in, h_out)
    assert torch.equal(dev, h_out)
    conv.forward_host(h_in, h_out)  # repeated calls reuse the plan's streams and events
    assert torch.equal(dev, h_out)


def test_argument_errors(sc):
    shp = datagen.C4B.with_batch(2)
    w, b = datagen.weights(shp)
    conv = make_conv(sc, shp, w, b)
    x = torch.zeros((3, shp.c, shp.h, shp.w), device=DEV)
    with pytest.raises(sc.SparseConvError) as e:      # n > max batch
        conv.forward(x)
    assert e.value.status == 1
    L = sc.lib()
    import ctypes
    out = torch.zeros((2,) + conv.out_shape, device=DEV)
    xs = torch.zeros(2 * shp.c * shp.h * shp.w + 1, device=DEV)
    st = L.sparse_conv_forward(conv._plan, 2, ctypes.c_void_p(xs.data_ptr() + 4), ctypes.c_void_p(out.data_ptr()), None)
    assert st == 1 and b"aligned" in L.sc_last_error()
    hx = torch.zeros(2 * shp.c * shp.h * shp.w)
    st = L.sparse_conv_forward(conv._plan, 2, ctypes.c_void_p(hx.data_ptr()), ctypes.c_void_p(out.data_ptr()), None)
    assert st == 1
    assert L.sparse_conv_forward(conv._plan, 0, ctypes.c_void_p(out.data_ptr()), ctypes.c_void_p(out.data_ptr()), None) == 1


def test_c5_chain_per_layer(sc):
    """C5 chain (R13/R14): each layer's oracle is fed the GPU's own input to
    that layer; lists bit-exact on that tensor; ReLU'd outputs compared with
    max(0, oracle).  Reduced batch (the full N=1024 chain is the bench's)."""
    n = 8
    layers = datagen.c5_weights()
    x = datagen.activations(datagen.C5_LAYERS[0].with_batch(n), datagen.C5_FIRST_SPARSITY)
    xd = torch.from_numpy(x).to(DEV)
    for li, (shp, (w, b)) in enumerate(zip(datagen.C5_LAYERS, layers)):
        shp = shp.with_batch(n)
        relu = li < 2
        conv = make_conv(sc, shp, w, b, relu=relu)
        out = conv.forward(xd)
        torch.cuda.synchronize()
        xin = xd.cpu().numpy()
        check_lists(conv, xin, n)
        check_conv(out.cpu().numpy(), xin, w, b, shp, relu=relu)
        if relu:
            s = 1.0 - float((out != 0).sum()) / out.numel()
            assert 0.9 < s < 0.99, s
        xd = out


# Every stage-2 kernel that matches a config: the generic kernel (0), the shipped variant,
# and the superseded round-1 tilings (tools/gen_gather.py SUPERSEDED: no longer built into the
# library), generated at run time through SC_JIT_FORCE="TY,KL,NW,MINB,CH,STAGES,SLOTS,PIECE".
JIT_TILINGS = {1: "7,2,7,1,8,4,3,254", 2: "3,2,7,1,8,4,3,254", 3: "2,2,7,1,4,4,3,254", 4: "2,2,7,1,4,4,3,254",
               5: "6,2,7,1,4,4,3,254", 28: "1,4,11,1,16,2,3,254", 29: "4,1,11,1,16,2,3,254",
               7: "7,1,11,1,16,4,3,254", 10: "3,3,11,1,8,4,3,254", 11: "3,4,7,1,8,3,3,254",
               12: "2,4,11,1,8,3,3,254", 13: "5,2,11,1,8,4,3,254", 14: "1,4,11,1,8,3,3,254",
               30: "2,1,11,1,16,2,3,254", 48: "3,3,11,1,16,2,2,254", 49: "2,4,11,1,16,3,3,510",
               50: "1,1,4,1,10,2,3,254"}
FORCED = ([("C2", v) for v in (0, 1, 7, 10, 11, 12, 13, 21)] + [("C4a", v) for v in (0, 2, 14, 28, 51)] +
          [("C4b", v) for v in (0, 4, 29, 30, 52)] + [("C3", v) for v in (0, 3, 33)] + [("C1", v) for v in (0, 5, 50, 57)])


def force_kernel(monkeypatch, variant):
    """Select stage-2 kernel `variant` for plans created from now on; returns the
    variant id the plan must report (-1 for a run-time generated tiling)."""
    if variant in JIT_TILINGS:
        monkeypatch.setenv("SC_JIT_FORCE", JIT_TILINGS[variant])
        return -1
    monkeypatch.setenv("SC_FORCE_VARIANT", str(variant))
    return variant


@pytest.mark.parametrize("cfg,variant", FORCED)
@pytest.mark.parametrize("s", [0.0, 0.95])
def test_forced_variants(sc, cfg, variant, s, monkeypatch):
    """Every stage-2 kernel that matches C2 / C4a / C4b / C3 against the oracle:
    tolerance on seeded data (dense s=0 too) and bit-exact on integer data."""
    want = force_kernel(monkeypatch, variant)
    shp = datagen.CONFIGS[cfg].with_batch(5)
    x = datagen.activations(shp, "channel" if (cfg == "C3" and s > 0) else s, seed=3)
    w, b = datagen.weights(shp, seed=3)
    conv = make_conv(sc, shp, w, b, max_batch=9)
    assert conv.variant[0] == want
    out = conv.forward(torch.from_numpy(x).to(DEV)).cpu().numpy()
    check_lists(conv, x, 5)
    check_conv(out, x, w, b, shp)
    xi, wi, bi = datagen.integer_case(shp, sparsity=0.7)
    conv = make_conv(sc, shp, wi, bi, max_batch=9)
    out = conv.forward(torch.from_numpy(xi).to(DEV)).cpu().numpy()
    ref, _ = oracle.conv_fp64(xi, wi, bi, shp.stride, shp.pad, shp.groups)
    assert np.array_equal(out.astype(np.float64), ref)
