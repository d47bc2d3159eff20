"""oracle -- TEST INFRASTRUCTURE ONLY (parity oracle for arXiv 1704.07724).

A plain, slow, obviously correct CPU implementation of what the hot path
computes.  Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import it.  It shares no code
with the CUDA path (``paper_1704_07724_b200``) and never imports it.

Every function cites the passage of /root/reference/PAPER.md ("P:<line>") it
follows; readings of garbled or silent passages are DESIGN.md R1..R18.

Functions
---------
output_shape        P:37 (Sec. 3, Table 1), floor form (R1)
conv_fp64           P:68-72 (Eq. 1) + stride/pad + batch/bias/groups
                    (R2-R4); fp64 accumulation, also returns the mass
                    sum |in|*|W| that scales the parity tolerance.  (C, OpenMP)
relu                P:74-78 (Eq. 2)
list_format         R9: row-tile height TH, index width, slot capacity
compact             P:123 (Sec. 4, ISC step 1) in the R9 list format  (C)
decompress          inverse of compact (for round-trip pins)
dense_macs          P:109 (Sec. 4): H_out*W_out*R*S*K*C per image (with groups:
                    C/G per output channel)
exact_nonzero_macs  P:121 (Sec. 4) "MACs can be reduce to rho*...": the exact
                    count = sum over nonzero inputs of Kg * covH(i) * covW(j),
                    the inverse map of P:121 with divisibility/range guards (R6)
estimated_macs      P:121: round(rho * dense_macs)
sparsity            P:121: 1 - #nonzeros / size

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
        lib.oracle_compact.restype = ctypes.c_int
        lib.oracle_compact.argtypes = [vp, i64, i64, i64, i64, i64, i64, i64, vp, vp, vp]
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


# --------------------------------------------------------------------------
# ISC step 1: nonzero compaction in the R9 list format
# --------------------------------------------------------------------------
def list_format(h, w):
    """DESIGN.md R9.  A list covers TH consecutive rows of one (n,c) plane:
    TH = H when H*W <= 256, else floor(256/W) rows (>= 1).  idx is u8 when
    TH*W <= 256 else u16.  Slot capacity = TH*W rounded up to 16 entries.
    Returns (TH, tiles_per_plane, idx_bytes, cap)."""
    if h * w <= 256:
        th = h
    else:
        th = max(1, 256 // w)
    idx_bytes = 1 if th * w <= 256 else 2
    cap = -(-(th * w) // 16) * 16
    tiles = -(-h // th)
    return th, tiles, idx_bytes, cap


def compact(x):
    """P:123 step 1.  x float32 [N][C][H][W] -> dict(values [L][cap] f32,
    idx [L][cap] u8/u16, counts [L] u32, th, tiles, idx_bytes, cap).
    Slack beyond counts[l] is left zero-filled here and is never compared."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    n, c, h, w = x.shape
    th, tiles, idx_bytes, cap = list_format(h, w)
    nl = n * c * tiles
    values = np.zeros((nl, cap), dtype=np.float32)
    idx = np.zeros((nl, cap), dtype=np.uint8 if idx_bytes == 1 else np.uint16)
    counts = np.zeros(nl, dtype=np.uint32)
    rc = _load().oracle_compact(_ptr(x), n, c, h, w, th, idx_bytes, cap,
                                _ptr(values), _ptr(idx), _ptr(counts))
    if rc != 0:
        raise ValueError("oracle_compact: invalid arguments")
    return dict(values=values, idx=idx, counts=counts, th=th, tiles=tiles,
                idx_bytes=idx_bytes, cap=cap)


def decompress(lists, shape):
    """Inverse of compact: scatter the entries back into a zero tensor."""
    n, c, h, w = shape
    th, tiles = lists["th"], lists["tiles"]
    out = np.zeros((n * c, h * w), dtype=np.float32)
    for l in range(n * c * tiles):
        plane, tile = divmod(l, tiles)
        cnt = int(lists["counts"][l])
        loc = lists["idx"][l, :cnt].astype(np.int64) + tile * th * w
        out[plane, loc] = lists["values"][l, :cnt]
    return out.reshape(n, c, h, w)


def tolerance_sparse(mass):
    """North star: |gpu - oracle| <= 1e-5 * mass + 1e-6 per element."""
    return 1e-5 * mass + 1e-6


def tolerance_dense_tf32(mass):
    """DESIGN.md R10: TF32 operands (RNA-rounded) cannot meet 1e-5*mass;
    the dense comparison path is checked at 2^-9 * mass + 1e-6."""
    return 2.0 ** -9 * mass + 1e-6
