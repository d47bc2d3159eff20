"""Seeded shape fuzz through the C ABI: shapes away from the BASELINE configs,
so that every fallback is exercised — the generic stage-2 kernel (widths with
no generated variant), the streamwise stage 1 (planes > 1024 elements or > 31
rows), strides 1-3, pads 0-3, groups 1-4, rectangular kernels, filter counts
that are not multiples of 32, one-pixel planes and outputs.

Per shape: stage-1 lists bit-exact against oracle.compact_lists (and the
streams against the test-side adapter's derivation from them); sparse
forward within the north-star bar 1e-5*mass + 1e-6; dense forward (where the
shape is supported) within the TF32 bar 2^-9*mass + 1e-6; integer data
bit-exact on both; backward (where supported) bit-exact on integer data."""
import numpy as np
import pytest
import torch

import oracle
from lists_check import check_plane_lists, check_streams
from paper_1704_07724_b200 import datagen

pytestmark = pytest.mark.gpu
DEV = torch.device("cuda:0")


@pytest.fixture(scope="module")
def sc():
    from paper_1704_07724_b200 import sparseconv
    sparseconv.lib()
    return sparseconv


def fuzz_shapes(count=24, seed=2024):
    rng = np.random.default_rng(seed)
    fixed = [  # hand-picked corners
        datagen.ConvShape("one_pixel", 900, 2, 3, 1, 1, 5, 1, 1, 1, 0, 1),          # 1x1 plane, 1x1 kernel
        datagen.ConvShape("kernel_eq_plane", 901, 2, 4, 5, 5, 7, 5, 5, 1, 0, 1),    # one output pixel
        datagen.ConvShape("big_pad", 902, 2, 3, 4, 4, 6, 3, 3, 1, 3, 1),            # pad > kernel/2
        datagen.ConvShape("large_plane", 903, 2, 6, 40, 36, 33, 3, 3, 1, 1, 1),     # streamwise stage 1
        datagen.ConvShape("tall_plane", 904, 2, 5, 48, 9, 17, 3, 3, 2, 1, 1),       # > 31 rows, stride 2
        datagen.ConvShape("rect_kernel", 905, 3, 8, 10, 12, 40, 3, 5, 1, 2, 2),     # R != S, groups 2
        datagen.ConvShape("stride3", 906, 2, 6, 17, 17, 20, 5, 5, 3, 2, 1),
        datagen.ConvShape("groups4", 907, 2, 16, 9, 9, 36, 3, 3, 1, 1, 4),
    ]
    out = list(fixed)
    for i in range(count - len(fixed)):
        groups = int(rng.choice([1, 1, 2, 3]))
        c = groups * int(rng.integers(1, 9))
        k = groups * int(rng.integers(1, 25))
        h, w = int(rng.integers(1, 30)), int(rng.integers(1, 30))
        stride = int(rng.choice([1, 1, 2, 3]))
        pad = int(rng.integers(0, 4))
        r = int(rng.integers(1, min(7, h + 2 * pad) + 1))
        s = int(rng.integers(1, min(7, w + 2 * pad) + 1))
        n = int(rng.integers(1, 5))
        out.append(datagen.ConvShape(f"rand{seed}_{i}", 910 + i, n, c, h, w, k, r, s, stride, pad, groups))
    return out


SHAPES = fuzz_shapes() + fuzz_shapes(count=32, seed=77)[8:]


def make_conv(sc, shp, w, b):
    return sc.SparseConv(torch.from_numpy(w).to(DEV), None if b is None else torch.from_numpy(b).to(DEV), shp.n,
                         shp.c, shp.h, shp.w, shp.stride, shp.pad, shp.groups)


@pytest.mark.parametrize("shp", SHAPES, ids=[s.name for s in SHAPES])
def test_fuzz_shape(sc, shp):
    x = datagen.activations(shp, 0.7, seed=5)
    w, b = datagen.weights(shp, seed=5)
    conv = make_conv(sc, shp, w, b)
    xd = torch.from_numpy(x).to(DEV)
    out = conv.forward(xd).cpu().numpy()
    # stage 1 bit-exact
    check_plane_lists(conv, x, shp.n)
    check_streams(conv, x, shp.n)
    # forward, sparse and dense
    ref, mass = oracle.conv_fp64(x, w, b, shp.stride, shp.pad, shp.groups)
    assert np.all(np.abs(out - ref) <= oracle.tolerance_sparse(mass)), conv.variant
    try:
        dense = conv.dense_forward(xd).cpu().numpy()
    except sc.SparseConvError:
        dense = None
    if dense is not None:
        assert np.all(np.abs(dense - ref) <= oracle.tolerance_dense_tf32(mass))
    # integer data: exact on every path
    xi, wi, bi = datagen.integer_case(shp, sparsity=0.6, seed=5)
    convi = make_conv(sc, shp, wi, bi)
    xid = torch.from_numpy(xi).to(DEV)
    refi, _ = oracle.conv_fp64(xi, wi, bi, shp.stride, shp.pad, shp.groups, want_mass=False)
    assert np.array_equal(convi.forward(xid).cpu().numpy().astype(np.float64), refi)
    if dense is not None:
        assert np.array_equal(convi.dense_forward(xid).cpu().numpy().astype(np.float64), refi)
    di = np.random.default_rng(5).integers(-3, 4, (shp.n, shp.k, shp.ho, shp.wo)).astype(np.float32)
    try:
        dw, db, dz = convi.backward(xid, torch.from_numpy(di).to(DEV))
    except sc.SparseConvError:
        return  # backward: plane-major shapes with 1x1 / 3x3 / 5x5 kernels only (documented)
    refb = oracle.conv_backward_fp64(xi, wi, di, shp.stride, shp.pad, shp.groups, want_mass=False)
    assert np.array_equal(dw.cpu().numpy().astype(np.float64), refb["dw"])
    assert np.array_equal(db.cpu().numpy().astype(np.float64), refb["dbias"])
    assert np.array_equal(dz.cpu().numpy().astype(np.float64), refb["dz"])


def test_too_large_is_unsupported(sc):
    """Element counts >= 2^31 are rejected before any allocation."""
    w = torch.zeros((8, 64, 3, 3), device=DEV)
    with pytest.raises(sc.SparseConvError) as e:
        sc.SparseConv(w, None, 2048, 64, 128, 128, pad=1)  # input 2048*64*128*128 = 2^31 elements
    assert e.value.status == 3  # SC_ERR_UNSUPPORTED


def chain_shapes():
    """Random 3-layer chains (layer l+1's input = layer l's output), ReLU fused between layers."""
    rng = np.random.default_rng(4242)
    chains = []
    for ci in range(6):
        n = int(rng.integers(1, 4))
        c, h, w = int(rng.integers(1, 40)), int(rng.integers(3, 16)), int(rng.integers(3, 30))
        layers = []
        fast = ci < 3  # widths with generated 3x3 kernels (V21 13, V44 14, V46 7): fused emission
        if fast:
            h = w = int([13, 14, 7][ci])
        for li in range(3):
            r = 3 if fast else int(rng.choice([1, 3, 5]))
            pad = 1 if fast else (r // 2 if rng.random() < 0.8 else 0)
            if r > h + 2 * pad or r > w + 2 * pad:
                r, pad = 1, 0
            k = int(rng.integers(1, 70))
            shp = datagen.ConvShape(f"chain{ci}_l{li}", 960 + 3 * ci + li, n, c, h, w, k, r, r, 1, pad, 1)
            layers.append(shp)
            c, h, w = k, shp.ho, shp.wo
        chains.append(layers)
    return chains


@pytest.mark.parametrize("ci", range(6))
@pytest.mark.parametrize("fused", [False, True])
def test_fuzz_chain(sc, ci, fused):
    """sparse_conv_forward_chain on random 3-layer chains, with materialised or (where the layer's
    kernel can emit lists) fused intermediates: the last output equals running the layers one by
    one through sparse_conv_forward, and every layer matches the oracle on its GPU input (R14)."""
    layers = chain_shapes()[ci]
    n = layers[0].n
    convs, ws = [], []
    for li, shp in enumerate(layers):
        w, b = datagen.weights(shp, seed=3, std=0.3)
        ws.append((w, b))
        convs.append(make_conv_relu(sc, shp, w, b, relu=li + 1 < len(layers)))
    x = torch.from_numpy(datagen.activations(layers[0], 0.8, seed=3)).to(DEV)
    outs = [torch.empty((n,) + c.out_shape, device=DEV) for c in convs]
    if fused:
        for li in range(len(convs) - 1):
            vid, name = convs[li].variant
            if vid > 0 and "_kl1" not in name:  # KL >= 2 fast kernels emit the next layer's lists
                outs[li] = None
    if fused and ci < 3:
        assert outs[0] is None and outs[1] is None, [c.variant for c in convs]
    sc.chain_forward(convs, x, outs)
    # layer by layer reference through the single-layer entry point
    cur = x
    for li, (conv, shp) in enumerate(zip(convs, layers)):
        y = conv.forward(cur)
        torch.cuda.synchronize()
        w, b = ws[li]
        ref, mass = oracle.conv_fp64(cur.cpu().numpy(), w, b, shp.stride, shp.pad, shp.groups)
        if li + 1 < len(layers):
            ref = np.maximum(ref, 0.0)
        assert np.all(np.abs(y.cpu().numpy() - ref) <= oracle.tolerance_sparse(mass)), f"layer {li}"
        if outs[li] is not None:
            assert torch.equal(outs[li], y), f"chain layer {li} differs from the single-layer forward"
        cur = y
    assert torch.equal(outs[-1], cur)


def make_conv_relu(sc, shp, w, b, relu):
    return sc.SparseConv(torch.from_numpy(w).to(DEV), torch.from_numpy(b).to(DEV), shp.n, shp.c, shp.h, shp.w,
                         shp.stride, shp.pad, shp.groups, fuse_relu=relu)


JIT_SHAPES = [  # no shipped variant: the plan generates one at creation (csrc/jit.cu)
    datagen.ConvShape("jit_w56_kl2", 980, 2, 8, 6, 56, 64, 3, 3, 1, 1, 1),
    datagen.ConvShape("jit_w20_kl4", 981, 2, 12, 20, 20, 130, 3, 3, 1, 1, 1),
    datagen.ConvShape("jit_s2_w32", 982, 2, 8, 32, 32, 100, 3, 3, 2, 1, 1),
    datagen.ConvShape("jit_1x1_w17", 983, 2, 40, 17, 17, 128, 1, 1, 1, 0, 1),
    datagen.ConvShape("jit_xpair_w12", 984, 3, 8, 10, 12, 20, 3, 5, 1, 2, 2),
    datagen.ConvShape("jit_kl3_w9", 985, 2, 16, 9, 9, 80, 5, 5, 1, 2, 1),
    # 1x1 with Kg >= 150: one-row tiles with the fewest k-blocks of KL = 4 / 6 / 8 (jit.cu choose())
    datagen.ConvShape("jit_1x1_w17_kl6", 986, 2, 40, 17, 17, 192, 1, 1, 1, 0, 1),
    datagen.ConvShape("jit_1x1_w10_kl8", 987, 2, 36, 10, 10, 256, 1, 1, 1, 0, 1),
    datagen.ConvShape("jit_1x1_w12_kl6_ragged", 988, 2, 30, 12, 12, 300, 1, 1, 1, 0, 1),
    datagen.ConvShape("jit_1x1_w20_kl4", 989, 2, 30, 20, 20, 256, 1, 1, 1, 0, 1),  # KL6/8 exceed 140 registers
]
JIT_EXPECT = {"jit_1x1_w17_kl6": "_ty1_kl6_", "jit_1x1_w10_kl8": "_ty1_kl8_", "jit_1x1_w12_kl6_ragged": "_ty1_kl6_",
              "jit_1x1_w20_kl4": "_kl4_"}


@pytest.mark.parametrize("shp", JIT_SHAPES, ids=[s.name for s in JIT_SHAPES])
def test_jit_variant(sc, shp):
    if not sc.lib().sc_jit_available():
        pytest.skip("NVRTC not loadable")
    x = datagen.activations(shp, 0.9, seed=8)
    w, b = datagen.weights(shp, seed=8)
    conv = make_conv(sc, shp, w, b)
    vid, name = conv.variant
    assert vid == -1 and name.startswith("jit_"), name
    assert JIT_EXPECT.get(shp.name, "") in name, name
    xd = torch.from_numpy(x).to(DEV)
    out = conv.forward(xd).cpu().numpy()
    ref, mass = oracle.conv_fp64(x, w, b, shp.stride, shp.pad, shp.groups)
    assert np.all(np.abs(out - ref) <= oracle.tolerance_sparse(mass))
    xi, wi, bi = datagen.integer_case(shp, sparsity=0.6, seed=8)
    refi, _ = oracle.conv_fp64(xi, wi, bi, shp.stride, shp.pad, shp.groups, want_mass=False)
    assert np.array_equal(make_conv(sc, shp, wi, bi).forward(torch.from_numpy(xi).to(DEV)).cpu().numpy(), refi)
    # the gated instantiation (device-side crossover) on the same plan
    for s_star, want in ((0.0, sc.SC_PATH_SPARSE), (1.0, sc.SC_PATH_DENSE)):
        conv.crossover = s_star
        try:
            o = conv.forward_auto(xd).cpu().numpy()
        except sc.SparseConvError:
            continue
        path, _ = conv.last_path()
        if path == sc.SC_PATH_SPARSE:
            assert np.all(np.abs(o - ref) <= oracle.tolerance_sparse(mass))
        else:
            assert np.all(np.abs(o - ref) <= oracle.tolerance_dense_tf32(mass))


def test_jit_force_rejects_invalid_parameters(sc, monkeypatch):
    """SC_JIT_FORCE sets outside the kernel's limits fail plan creation (SC_ERR_UNSUPPORTED)
    instead of running: 64 weight chunks of 16 channels (Cg = 1024), KL = 5 (no packing)."""
    if not sc.lib().sc_jit_available():
        pytest.skip("NVRTC not loadable")
    shp = datagen.ConvShape("force_bad", 990, 1, 1024, 7, 7, 64, 1, 1, 1, 0, 1)
    w, b = datagen.weights(shp)
    for force, why in (("2,4,11,1,16,2,3,254", "63 weight chunks"), ("1,5,11,1,32,2,3,254", "KL must be")):
        monkeypatch.setenv("SC_JIT_FORCE", force)
        with pytest.raises(sc.SparseConvError) as e:
            make_conv(sc, shp, w, b)
        assert e.value.status == 3 and why in str(e.value), str(e.value)
    monkeypatch.setenv("SC_JIT_FORCE", "2,4,11,1,17,2,3,254")  # 61 chunks: accepted
    assert make_conv(sc, shp, w, b).variant[0] == -1
