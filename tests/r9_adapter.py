"""Test-side adapter: the stage-2 kernel's instruction-stream format (DESIGN.md
reading R9) derived from the paper-level step-1 lists of the oracle.

The oracle (oracle.compact_lists) computes only what the paper states for ISC
step 1 (Sec. 4): per (image, channel, row tile) the nonzero
values with their row and column.  How the CUDA path regroups those entries
for its stage-2 interpreter -- one stream per (image, output row tile of TY
rows), input windows with halo rows duplicated between neighbouring tiles,
a per-channel marker whose code carries the filter rows the channel reaches --
is a kernel design choice, not the method.  It lives here, in tests/, so that
the oracle never restates the kernel's format.  Pins: tests/test_r9_adapter.py
(decompression round trip, the marker-mask property in the forward-index form
of Eq. 1, the hand-worked golden stream).

R9: tile t covers output rows [t*TY, (t+1)*TY); its input window is
NWR = (TY-1)*T + R rows starting at i_lo = t*TY*T - P, all W columns,
NWIN = NWR*W positions.  Stream (n, t) = for every channel c (ascending) with
at least one entry inside the window: a marker (c, NWIN + mask), then those
entries (bits(x), (i - i_lo)*W + j) in row-major order; bit r of mask is set
iff some entry sits at a window row wi with wi - r = ty*T, 0 <= ty < TY.
offs[n][t][c] = index of c's marker (== offs[n][t][c+1] when it has none),
offs[n][t][C] = stream length.
"""
from __future__ import annotations

import numpy as np


def stream_format(c, h, w, r, stride, pad, ty, ho):
    """R9 geometry: (tiles, NWR, NWIN, stream capacity).  Capacity = C markers
    + every in-plane window position, rounded up to an even entry count."""
    tiles = -(-ho // ty)
    nwr = (ty - 1) * stride + r
    nwin = nwr * w
    cap = c * (1 + min(nwr, h) * w)
    cap += cap & 1
    return tiles, nwr, nwin, cap


def _live_entries(lists):
    """Flatten the oracle lists to per-entry arrays (n, c, i, j, bits), sorted
    by (n, c, i, j) -- the lists are row-major per (n, c, row tile)."""
    cnt = lists["counts"].astype(np.int64)
    k = np.arange(lists["values"].shape[-1])
    live = k[None, None, None, :] < cnt[..., None]
    n_e, c_e, _, _ = np.nonzero(live)
    return (n_e.astype(np.int64), c_e.astype(np.int64), lists["rows"][live].astype(np.int64),
            lists["cols"][live].astype(np.int64), lists["values"][live].astype(np.uint32))


def streams_from_lists(lists, shape, r, stride, pad, ty):
    """R9 streams of a batch from oracle.compact_lists output.  Returns
    dict(entries u32 [N][tiles][cap][2], offs u32 [N][tiles][C+1], tiles, nwr,
    nwin, cap, ty); entries beyond each stream's length are zero."""
    n, c, h, w = shape
    ho = (h + 2 * pad - r) // stride + 1
    tiles, nwr, nwin, cap = stream_format(c, h, w, r, stride, pad, ty, ho)
    n_e, c_e, i_e, j_e, v_e = _live_entries(lists)
    entries = np.zeros((n, tiles, cap, 2), np.uint32)
    offs = np.zeros((n, tiles, c + 1), np.uint32)
    for t in range(tiles):
        i_lo = t * ty * stride - pad
        sel = (i_e >= i_lo) & (i_e < i_lo + nwr)
        ns, cs, wi, js, vs = n_e[sel], c_e[sel], i_e[sel] - i_lo, j_e[sel], v_e[sel]
        g = ns * c + cs                                   # group id, ascending (sorted input)
        cnt = np.bincount(g, minlength=n * c).reshape(n, c)
        size = cnt + (cnt > 0)                            # marker only with entries
        start = np.cumsum(size, axis=1) - size            # exclusive, per image
        offs[:, t, :c] = start
        offs[:, t, c] = size.sum(axis=1)
        if len(g) == 0:
            continue
        first = np.searchsorted(g, g, side="left")        # first entry index of each group
        rank = np.arange(len(g)) - first
        pos = start[ns, cs] + 1 + rank
        entries[ns, t, pos, 0] = vs
        entries[ns, t, pos, 1] = wi * w + js
        # marker: filter rows reached (wi - rr = ty'*stride, 0 <= ty' < ty)
        bits = np.zeros(len(g), np.int64)
        for rr in range(r):
            d = wi - rr
            bits |= ((d >= 0) & (d % stride == 0) & (d // stride < ty)).astype(np.int64) << rr
        gstart = np.flatnonzero(np.r_[True, g[1:] != g[:-1]])
        mask = np.bitwise_or.reduceat(bits, gstart)
        gn, gc = ns[gstart], cs[gstart]
        mpos = start[gn, gc]
        entries[gn, t, mpos, 0] = gc
        entries[gn, t, mpos, 1] = nwin + mask
    return dict(entries=entries, offs=offs, tiles=tiles, nwr=nwr, nwin=nwin, cap=cap, ty=ty)


def decompress_streams(st, shape, stride, pad):
    """Scatter every stream's entries back into a zero tensor (inputs inside
    several windows are written more than once, with the same bits); checks
    that each non-empty channel range starts with its marker."""
    n, c, h, w = shape
    out = np.zeros(shape, dtype=np.float32).reshape(n, c, h * w).view(np.uint32)
    for ni in range(n):
        for t in range(st["tiles"]):
            i_lo = t * st["ty"] * stride - pad
            e = st["entries"][ni, t]
            of = st["offs"][ni, t]
            for ci in range(c):
                a, b = int(of[ci]), int(of[ci + 1])
                if a == b:
                    continue
                assert b > a + 1 and e[a, 0] == ci and e[a, 1] >= st["nwin"], "bad channel marker"
                code = e[a + 1:b, 1].astype(np.int64)
                rows = i_lo + code // w
                out[ni, ci, rows * w + code % w] = e[a + 1:b, 0]
    return out.view(np.float32).reshape(shape)
