"""C5 (BASELINE.json configs[4]): AlexNet conv3 -> ReLU -> conv4 -> ReLU ->
conv5 through the C-ABI library with ReLU fused into the epilogue (Eq. 2,
PAPER.md:77; reading R15).  Parity per layer on the GPU's own input to that
layer (reading R14): a ReLU threshold near 0 can flip between fp32 and fp64,
so each layer's oracle sees exactly the tensor the GPU layer saw; ReLU'd
outputs are compared with max(0, oracle) (max is 1-Lipschitz, the tolerance
carries over).  Stage-1 lists are checked bit-exactly on the same tensors."""
import numpy as np
import pytest
import torch

import oracle
from paper_1704_07724_b200 import datagen
from lists_check import check_plane_lists, check_streams

pytestmark = pytest.mark.gpu
DEV = torch.device("cuda:0")


def run_chain(n, images):
    from paper_1704_07724_b200 import sparseconv as sc
    layers = [shp.with_batch(n) for shp in datagen.C5_LAYERS]
    weights = datagen.c5_weights()
    x = torch.from_numpy(datagen.activations(layers[0], datagen.C5_FIRST_SPARSITY)).to(DEV)
    worst = 0.0
    for li, shp in enumerate(layers):
        w, b = weights[li]
        relu = li + 1 < len(layers)
        conv = sc.SparseConv(torch.from_numpy(w).to(DEV), torch.from_numpy(b).to(DEV), n, shp.c, shp.h, shp.w,
                             shp.stride, shp.pad, shp.groups, fuse_relu=relu)
        y = conv.forward(x)
        torch.cuda.synchronize()
        xin = x.cpu().numpy()
        assert check_plane_lists(conv, xin, n), f"layer {li}: no plane lists"
        check_streams(conv, xin, n)
        got = y.cpu().numpy()
        for i in images:
            ref, mass = oracle.conv_fp64(xin[i:i + 1], w, b, shp.stride, shp.pad, shp.groups)
            if relu:
                ref = np.maximum(ref, 0.0)
            err = np.abs(got[i:i + 1].astype(np.float64) - ref) / oracle.tolerance_sparse(mass)
            assert err.max() <= 1.0, f"layer {li} image {i}: max err/tol {err.max():.3f}"
            worst = max(worst, float(err.max()))
        if relu:
            s_next = 1.0 - float((y != 0).sum().item()) / y.numel()
            assert 0.85 < s_next < 0.995, f"layer {li} output sparsity {s_next}"   # R13 bias shift holds s~0.95
        x = y
    return worst


def test_c5_chain_small_batch_all_images():
    run_chain(4, range(4))


def test_c5_chain_full_batch_sampled_images():
    run_chain(1024, [0, 511, 1023])


def _chain_setup(n):
    from paper_1704_07724_b200 import sparseconv as sc
    layers = [shp.with_batch(n) for shp in datagen.C5_LAYERS]
    weights = datagen.c5_weights()
    convs = []
    for li, shp in enumerate(layers):
        w, b = weights[li]
        convs.append(sc.SparseConv(torch.from_numpy(w).to(DEV), torch.from_numpy(b).to(DEV), n, shp.c, shp.h, shp.w,
                                   shp.stride, shp.pad, shp.groups, fuse_relu=li + 1 < len(layers)))
    x = torch.from_numpy(datagen.activations(layers[0], datagen.C5_FIRST_SPARSITY)).to(DEV)
    return sc, layers, weights, convs, x


@pytest.mark.parametrize("n", [3, 64, 260, 512])  # n >= 256: chunks of images on two streams
def test_chain_fused_lists_match_compaction_and_oracle(n):
    """f1: intermediate layers emit the next layer's stage-1 lists from
    their epilogue.  With the intermediate outputs also materialised, every
    consumer's paper-level lists must equal oracle.compact_lists of the
    producer's output bit for bit (and its R9 streams the adapter's derivation), and every layer must meet the tolerance on its own
    input (R14); without them the final output must be bit-identical."""
    sc, layers, weights, convs, x = _chain_setup(n)
    outs = [torch.empty((n,) + c.out_shape, device=DEV) for c in convs]
    sc.chain_forward(convs, x, outs)
    torch.cuda.synchronize()
    inputs = [x] + outs[:-1]
    for li, (shp, conv) in enumerate(zip(layers, convs)):
        xin = inputs[li].cpu().numpy()
        # layer 0: lists of the input tensor (layout 1); later layers: the per-row lists the
        # producer's epilogue emitted (layout 2) -- both against the oracle's lists of the
        # materialised producer output
        assert check_plane_lists(conv, xin, n), f"layer {li}: no plane lists"
        assert conv.plane_lists(n)["layout"] == (1 if li == 0 else 2)
        check_streams(conv, xin, n)
        w, b = weights[li]
        got = outs[li].cpu().numpy()
        for i in sorted({0, n - 1}):
            ref, mass = oracle.conv_fp64(xin[i:i + 1], w, b, shp.stride, shp.pad, shp.groups)
            if li + 1 < len(layers):
                ref = np.maximum(ref, 0.0)
            err = np.abs(got[i:i + 1].astype(np.float64) - ref) / oracle.tolerance_sparse(mass)
            assert err.max() <= 1.0, f"layer {li} image {i}: max err/tol {err.max():.3f}"
    # fused only: no intermediate dense tensors, same final bits
    fin = torch.empty_like(outs[-1])
    sc.chain_forward(convs, x, [None] * (len(convs) - 1) + [fin])
    torch.cuda.synchronize()
    assert torch.equal(fin, outs[-1])


def test_chunked_chain_first_call_under_capture():
    """n >= 256 runs the chain in two image chunks on plan-owned streams, created on the first call
    made outside stream capture; a first call under capture runs unchunked.  Both give the same
    bits, and a graph captured later (chunked, forked onto the plan's streams) replays them."""
    n = 260
    sc, layers, weights, convs, x = _chain_setup(n)
    fin = torch.empty((n,) + convs[-1].out_shape, device=DEV)
    s = torch.cuda.Stream()
    outs = [None] * (len(convs) - 1) + [fin]
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        sc.chain_forward(convs, x, outs, stream=s)
    g.replay()
    torch.cuda.synchronize()
    captured = fin.clone()
    fin.zero_()
    sc.chain_forward(convs, x, outs)  # eager: creates the streams, chunked
    torch.cuda.synchronize()
    assert torch.equal(fin, captured)
    g2 = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g2, stream=s):
        sc.chain_forward(convs, x, outs, stream=s)
    fin.zero_()
    g2.replay()
    torch.cuda.synchronize()
    assert torch.equal(fin, captured)
