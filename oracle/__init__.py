"""oracle -- TEST INFRASTRUCTURE ONLY (parity oracle for arXiv 1704.07724).

A plain, slow, obviously correct CPU implementation of what the hot path
computes.  Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import it.  It shares no code
with the CUDA path (``paper_1704_07724_b200``) and never imports it.

Every function cites the passage of /root/reference/PAPER.md ("P:<line>") it
follows; readings of garbled or silent passages are DESIGN.md R1..R20.
The stage-2 kernel's instruction-stream format (R9) is NOT computed here: it
is an implementation detail of the CUDA path, derived from compact_lists by
the test-side adapter tests/r9_adapter.py.

Functions
---------
output_shape        P:37 (Sec. 3, Table 1), floor form (R1)
conv_fp64           P:68-72 (Eq. 1) + stride/pad + batch/bias/groups
                    (R2-R4); fp64 accumulation, also returns the mass
                    sum |in|*|W| that scales the parity tolerance.  (C, OpenMP)
relu                P:74-78 (Eq. 2)
list_rows           SURVEY 8c item 9: rows per list (whole plane if H*W <= 256)
compact_lists       P:123 (Sec. 4, ISC step 1): per (image, channel, row tile)
                    the nonzero values with their row and column, row-major (C)
decompress_lists    inverse of compact_lists (for round-trip pins)
dense_macs          P:109 (Sec. 4): H_out*W_out*R*S*K*C per image (with groups:
                    C/G per output channel)
exact_nonzero_macs  P:121 (Sec. 4) "MACs can be reduce to rho*...": the exact
                    count = sum over nonzero inputs of Kg * covH(i) * covW(j),
                    the inverse map of P:121 with divisibility/range guards (R6)
estimated_macs      P:121: round(rho * dense_macs)
sparsity            P:121: 1 - #nonzeros / size
conv_backward_fp64  SURVEY 8f row f4 (training): weight gradient,
                    bias gradient and the input gradient through the producing
                    ReLU (Eq. 2), R19-R20.  (C, OpenMP)

Parity status: every function above is pinned by tests/test_oracle.py (brute
force with exact rationals, torch conv2d float64, closed forms, invariants,
tests/golden fixtures).  No function is "parity unpinned".
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None


def build(force: bool = False) -> str:
    """Compile oracle.c -> liboracle.so (plain gcc -O2 -fopenmp, no fast-math)."""
    src = os.path.join(_HERE, "oracle.c")
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(src):
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-std=c11",
                               "-fno-fast-math", "-ffp-contract=off",
                               src, "-o", _LIB_PATH, "-lm"])
    return _LIB_PATH


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB_PATH)
        i64 = ctypes.c_int64
        vp = ctypes.c_void_p
        lib.oracle_conv_fp64.restype = ctypes.c_int
        lib.oracle_conv_fp64.argtypes = [vp, vp, vp] + [i64] * 10 + [vp, vp]
        lib.oracle_conv_backward_fp64.restype = ctypes.c_int
        lib.oracle_conv_backward_fp64.argtypes = [vp, vp, vp] + [i64] * 10 + [vp] * 5
        lib.oracle_compact_lists.restype = ctypes.c_int
        lib.oracle_compact_lists.argtypes = [vp] + [i64] * 5 + [vp] * 4
        _lib = lib
    return _lib


def _ptr(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


# --------------------------------------------------------------------------
# Shapes and counts
# --------------------------------------------------------------------------
def output_shape(n, c, h, w, k, r, s, stride=1, pad=0, groups=1):
    """P:37 gives H_out=(H+2P-R+1)/T, non-integral for LeNet-Conv2;
    R1 reading: floor((H+2P-R)/T)+1 (equal at T=1).  Returns (N, K, Ho, Wo)."""
    if min(n, c, h, w, k, r, s, stride, groups) < 1 or pad < 0:
        raise ValueError("extents must be >= 1 and pad >= 0")
    if c % groups or k % groups:
        raise ValueError("groups must divide C and K")
    if r > h + 2 * pad or s > w + 2 * pad:
        raise ValueError("kernel larger than padded input")
    return (n, k, (h + 2 * pad - r) // stride + 1, (w + 2 * pad - s) // stride + 1)


def dense_macs(n, c, h, w, k, r, s, stride=1, pad=0, groups=1):
    """a direct convolution takes H_out*W_out*R*S*K*C MACs per image
    (each output channel reads C/G input channels with groups)."""
    _, _, ho, wo = output_shape(n, c, h, w, k, r, s, stride, pad, groups)
    return n * ho * wo * r * s * k * (c // groups)


def _coverage(i, extent_in, kk, stride, pad, extent_out):
    """Number of taps r<kk for which input row i maps to a valid output row:
    y = (i + P - r)/T integral and 0 <= y < extent_out  (inverse map, R6)."""
    cnt = 0
    for r in range(kk):
        num = i + pad - r
        if num >= 0 and num % stride == 0 and num // stride < extent_out:
            cnt += 1
    return cnt


def exact_nonzero_macs(x, k, r, s, stride=1, pad=0, groups=1):
    """with zero inputs skipped, each nonzero input (n,c,i,j) performs
    Kg * covH(i) * covW(j) MACs.  x: float32 [N][C][H][W]."""
    n, c, h, w = x.shape
    _, _, ho, wo = output_shape(n, c, h, w, k, r, s, stride, pad, groups)
    cov_h = np.array([_coverage(i, h, r, stride, pad, ho) for i in range(h)], dtype=np.int64)
    cov_w = np.array([_coverage(j, w, s, stride, pad, wo) for j in range(w)], dtype=np.int64)
    nz = (x != 0).astype(np.int64)                      # IEEE compare, -0.0 is zero
    per_pos = nz.sum(axis=(0, 1))                       # [H][W] nonzero counts
    return int((k // groups) * (cov_h[:, None] * cov_w[None, :] * per_pos).sum())


def estimated_macs(x, k, r, s, stride=1, pad=0, groups=1):
    """rho * H_out*W_out*R*S*K*C with rho = #nonzeros/(C*H*W)."""
    n, c, h, w = x.shape
    rho = np.count_nonzero(x) / x.size
    return int(round(rho * dense_macs(n, c, h, w, k, r, s, stride, pad, groups)))


def sparsity(x):
    """sparsity = 1 - rho, rho = #nonzeros / size (exact zero test)."""
    return 1.0 - np.count_nonzero(x) / x.size


def relu(x):
    """P:77, Eq. 2: Z = max(0, O)."""
    return np.maximum(x, np.zeros((), dtype=x.dtype))


# --------------------------------------------------------------------------
# The convolution (Eq. 1)
# --------------------------------------------------------------------------
def conv_fp64(x, w, bias=None, stride=1, pad=0, groups=1, want_mass=True):
    """P:68-72 Eq. 1 with stride T and padding P, batch, bias, groups.

    out[n,k,y,x] = bias[k] + sum_{c,r,t} in[n,c,yT+r-P,xT+t-P] * W[k,c,r,t]
    computed in double by the C 7-loop in oracle.c.  Returns (out, mass) as
    float64 arrays [N][K][Ho][Wo] (mass None if not requested)."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    w = np.ascontiguousarray(w, dtype=np.float32)
    n, c, h, ww = x.shape
    k, cg, r, s = w.shape
    if cg * groups != c:
        raise ValueError("weight shape does not match C/groups")
    shp = output_shape(n, c, h, ww, k, r, s, stride, pad, groups)
    b = None if bias is None else np.ascontiguousarray(bias, dtype=np.float32)
    out = np.empty(shp, dtype=np.float64)
    mass = np.empty(shp, dtype=np.float64) if want_mass else None
    rc = _load().oracle_conv_fp64(_ptr(x), _ptr(w), _ptr(b), n, c, h, ww, k, r, s,
                                  stride, pad, groups, _ptr(out), _ptr(mass))
    if rc != 0:
        raise ValueError("oracle_conv_fp64: invalid shape")
    return out, mass


def conv_backward_fp64(x, w, dout, stride=1, pad=0, groups=1, want_mass=True):
    """Gradients of Eq. 1 (R19-R20), in double.

    dw[k,c,r,t] = sum_{n,y,x} in[n,c,yT+r-P,xT+t-P] * dout[n,k,y,x]
    dbias[k]    = sum_{n,y,x} dout[n,k,y,x]
    dz[n,c,i,j] = [in != 0] * sum_{k,r,t} W[k,c,r,t] * dout[n,k,(i+P-r)/T,(j+P-t)/T]
                  (terms with a non-integral or out-of-range output index dropped)
    dz is the gradient through the ReLU that produced `in` (Eq. 2).  Returns
    dict(dw, dw_mass, dbias, dz, dz_mass) of float64 arrays (masses None if not
    requested)."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    w = np.ascontiguousarray(w, dtype=np.float32)
    dout = np.ascontiguousarray(dout, dtype=np.float32)
    n, c, h, ww = x.shape
    k, cg, r, s = w.shape
    if cg * groups != c:
        raise ValueError("weight shape does not match C/groups")
    shp = output_shape(n, c, h, ww, k, r, s, stride, pad, groups)
    if dout.shape != shp:
        raise ValueError(f"dout shape {dout.shape} != output shape {shp}")
    dw = np.empty(w.shape, np.float64)
    dbias = np.empty(k, np.float64)
    dz = np.empty(x.shape, np.float64)
    dwm = np.empty(w.shape, np.float64) if want_mass else None
    dzm = np.empty(x.shape, np.float64) if want_mass else None
    rc = _load().oracle_conv_backward_fp64(_ptr(x), _ptr(w), _ptr(dout), n, c, h, ww, k, r, s, stride, pad,
                                           groups, _ptr(dw), _ptr(dwm), _ptr(dbias), _ptr(dz), _ptr(dzm))
    if rc != 0:
        raise ValueError("oracle_conv_backward_fp64: invalid shape")
    return dict(dw=dw, dw_mass=dwm, dbias=dbias, dz=dz, dz_mass=dzm)


# --------------------------------------------------------------------------
# ISC step 1: nonzero compaction as the paper states it
# --------------------------------------------------------------------------
def list_rows(h, w):
    """SURVEY 8c item 9 (the north star leaves "row-tile" open): a list covers
    TH consecutive input rows of one (image, channel) plane -- the whole plane
    when H*W <= 256, else the most rows with TH*W <= 256, at least 1.
    Returns (TH, tiles per plane, index bytes: 1 if TH*W <= 256 else 2)."""
    if h < 1 or w < 1:
        raise ValueError("extents must be >= 1")
    th = h if h * w <= 256 else max(1, 256 // w)
    return th, -(-h // th), 1 if th * w <= 256 else 2


def compact_lists(x, th=None):
    """P:123 step 1: "skip all the zero elements of the input data, and store
    the non-zero values in a vector with their column and row information".

    x float32 [N][C][H][W].  One list per (n, c, row tile t) of TH rows
    (default: list_rows(H, W)); entries in row-major scan order, zero test
    x != 0.0f (R7).  Returns dict(values u32, rows i32, cols i32 each
    [N][C][tiles][TH*W] (slots at or beyond the count are zero and never
    compared), counts u32 [N][C][tiles], th, tiles).  (C, oracle.c)"""
    x = np.ascontiguousarray(x, dtype=np.float32)
    n, c, h, w = x.shape
    if th is None:
        th = list_rows(h, w)[0]
    if th < 1:
        raise ValueError("th must be >= 1")
    tiles = -(-h // th)
    values = np.zeros((n, c, tiles, th * w), np.uint32)
    rows = np.zeros((n, c, tiles, th * w), np.int32)
    cols = np.zeros((n, c, tiles, th * w), np.int32)
    counts = np.zeros((n, c, tiles), np.uint32)
    rc = _load().oracle_compact_lists(_ptr(x), n, c, h, w, th, _ptr(values), _ptr(rows), _ptr(cols), _ptr(counts))
    if rc != 0:
        raise ValueError("oracle_compact_lists: invalid arguments")
    return dict(values=values, rows=rows, cols=cols, counts=counts, th=th, tiles=tiles)


def decompress_lists(lists, shape):
    """Inverse of compact_lists: scatter every list's (row, col, value) back
    into a zero tensor of `shape` (used by the round-trip pins)."""
    n, c, h, w = shape
    out = np.zeros(shape, np.float32).view(np.uint32)
    cnt = lists["counts"].astype(np.int64)
    k = np.arange(lists["values"].shape[-1])
    live = k[None, None, None, :] < cnt[..., None]
    ni, ci, _, ki = np.nonzero(live)
    out[ni, ci, lists["rows"][live], lists["cols"][live]] = lists["values"][live]
    return out.view(np.float32)


def tolerance_sparse(mass):
    """North star: |gpu - oracle| <= 1e-5 * mass + 1e-6 per element."""
    return 1e-5 * mass + 1e-6


def tolerance_dense_tf32(mass):
    """DESIGN.md R10: TF32 operands (RNA-rounded) cannot meet 1e-5*mass;
    the dense comparison path is checked at 2^-9 * mass + 1e-6."""
    return 2.0 ** -9 * mass + 1e-6
