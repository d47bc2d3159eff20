"""Pins for the test-side adapter (tests/r9_adapter.py) that derives the
stage-2 kernel's stream format (R9) from the oracle's paper-level
step-1 lists.  Checked against things other than the adapter itself:
np.nonzero of each input window, the decompression round trip, the marker
mask stated in the forward-index form of Eq. 1 (output row y reads
input row y*T + r - P), and a hand-worked golden stream.  CPU only."""
import numpy as np
import pytest

import oracle
import r9_adapter
from conftest import read_golden_kv


def test_stream_format():
    # (c, h, w, r, stride, pad, ty, ho) -> (tiles, nwr, nwin, cap)
    assert r9_adapter.stream_format(256, 13, 13, 3, 1, 1, 13, 13) == (1, 15, 195, 256 * (1 + 13 * 13))
    assert r9_adapter.stream_format(256, 13, 13, 3, 1, 1, 7, 13) == (2, 9, 117, 256 * (1 + 9 * 13))
    assert r9_adapter.stream_format(20, 11, 11, 5, 2, 1, 5, 5) == (1, 13, 143, 20 * (1 + 11 * 11))
    assert r9_adapter.stream_format(3, 5, 5, 1, 1, 0, 2, 5) == (3, 2, 10, 3 * 11 + 1)


def _streams(x, r, stride, pad, ty, th=None):
    return r9_adapter.streams_from_lists(oracle.compact_lists(x, th), x.shape, r, stride, pad, ty)


def test_hand_worked_stream():
    g = read_golden_kv("hand_example_3x3.txt")
    x = np.array(g["input"], dtype=np.float32).reshape(1, 1, 3, 3)
    st = _streams(x, 3, 1, 1, 3)
    assert st["tiles"] == 1 and st["nwin"] == 15
    assert list(st["offs"][0, 0]) == [int(v) for v in g["stream_offs"]]
    e = st["entries"][0, 0, :3]
    a = [int(g["stream_a"][0])] + [int(np.float32(v).view(np.uint32)) for v in g["stream_a"][1:]]
    assert list(e[:, 0]) == a
    assert list(e[:, 1]) == [int(v) for v in g["stream_b"]]


def _window_entries_reference(x, r, stride, pad, ty):
    """np.nonzero of each (image, tile, channel) input window, row-major."""
    n, c, h, w = x.shape
    ho = (h + 2 * pad - r) // stride + 1
    tiles = -(-ho // ty)
    nwr = (ty - 1) * stride + r
    out = {}
    for ni in range(n):
        for t in range(tiles):
            i_lo = t * ty * stride - pad
            rows = [i for i in range(i_lo, i_lo + nwr) if 0 <= i < h]
            for ci in range(c):
                if rows:
                    sub = x[ni, ci, rows[0]:rows[-1] + 1]
                    ii, jj = np.nonzero(sub)
                    vals = sub[ii, jj].view(np.uint32)
                    codes = (ii + rows[0] - i_lo) * w + jj
                else:
                    vals = codes = np.zeros(0, np.int64)
                out[(ni, t, ci)] = (vals.astype(np.uint32), codes.astype(np.uint32))
    return out, tiles, nwr * w


def _mask_forward_index(x, ni, ci, t, r, stride, pad, ty, ho):
    """Bit rr set iff filter row rr, applied at some output row y of tile t
    (y = t*TY + ty' < H_out, Eq. 1 forward index i = y*T + rr - P), reads a
    nonzero input row of channel ci."""
    h = x.shape[2]
    m = 0
    for rr in range(r):
        for tyq in range(ty):
            i = (t * ty + tyq) * stride + rr - pad
            if 0 <= i < h and np.any(x[ni, ci, i] != 0):
                m |= 1 << rr
    return m


CASES = [((2, 3, 13, 13), 3, 1, 1, 13), ((2, 3, 13, 13), 3, 1, 1, 7), ((2, 4, 13, 13), 3, 1, 1, 2),
         ((1, 2, 28, 28), 3, 1, 1, 3), ((2, 2, 27, 27), 5, 1, 2, 2), ((1, 4, 11, 11), 5, 2, 1, 5),
         ((2, 3, 7, 7), 1, 1, 0, 3), ((3, 2, 1, 1), 1, 1, 0, 1), ((2, 3, 12, 12), 5, 1, 0, 4)]


@pytest.mark.parametrize("shape,r,stride,pad,ty", CASES)
@pytest.mark.parametrize("density", [0.15, 0.03])
def test_streams_against_numpy_windows_and_roundtrip(shape, r, stride, pad, ty, density):
    rng = np.random.default_rng(sum(shape) + ty + int(density * 100))
    x = (np.abs(rng.standard_normal(shape)) * (rng.random(shape) < density)).astype(np.float32)
    st = _streams(x, r, stride, pad, ty)
    ref, tiles, nwin = _window_entries_reference(x, r, stride, pad, ty)
    ho = (shape[2] + 2 * pad - r) // stride + 1
    assert st["tiles"] == tiles and st["nwin"] == nwin
    n, c = shape[:2]
    for ni in range(n):
        for t in range(tiles):
            of = st["offs"][ni, t].astype(np.int64)
            e = st["entries"][ni, t]
            for ci in range(c):
                a, b = of[ci], of[ci + 1]
                vals, codes = ref[(ni, t, ci)]
                if len(vals) == 0:
                    assert a == b  # no entry in the window: no marker (R9)
                    continue
                assert e[a, 0] == ci
                assert e[a, 1] == nwin + _mask_forward_index(x, ni, ci, t, r, stride, pad, ty, ho)
                assert np.array_equal(e[a + 1:b, 0], vals)
                assert np.array_equal(e[a + 1:b, 1], codes)
            assert of[c] <= st["cap"]
    back = r9_adapter.decompress_streams(st, shape, stride, pad)
    covered = np.zeros(shape[2], bool)
    for t in range(tiles):
        lo = t * ty * stride - pad
        covered[max(lo, 0):max(min(lo + (ty - 1) * stride + r, shape[2]), 0)] = True
    assert np.array_equal(back[:, :, covered].view(np.uint32), x[:, :, covered].view(np.uint32))


def test_streams_independent_of_list_row_tiling():
    """The streams depend on the input only, not on how the oracle's lists are cut into row tiles."""
    rng = np.random.default_rng(5)
    x = (rng.random((2, 3, 28, 28)) * (rng.random((2, 3, 28, 28)) < 0.1)).astype(np.float32)
    a = _streams(x, 3, 1, 1, 2, th=None)
    for th in (1, 5, 28):
        b = _streams(x, 3, 1, 1, 2, th=th)
        assert np.array_equal(a["offs"], b["offs"]) and np.array_equal(a["entries"], b["entries"])


def test_empty_channels_have_no_marker():
    """R9: a channel with no nonzero inside a tile's window contributes nothing to that
    tile's stream (offs[c] == offs[c+1]); the others keep marker + entries in order."""
    x = np.zeros((1, 3, 6, 4), np.float32)
    x[0, 0, 0, 1] = 1.0      # only in tile 0's window (rows -1..2 with ty=2, r=3, pad=1)
    x[0, 2, 5, 2] = 2.0      # only in the last tile's window
    st = _streams(x, 3, 1, 1, 2)
    assert st["tiles"] == 3
    of = st["offs"][0].astype(np.int64)
    e = st["entries"][0]
    assert list(of[0]) == [0, 2, 2, 2]             # tile 0: channel 0 only
    assert e[0, 0, 0] == 0 and e[0, 1, 1] == 1 * 4 + 1
    assert list(of[1]) == [0, 0, 0, 0]             # tile 1 (rows 1..4): empty stream
    assert list(of[2]) == [0, 0, 0, 2]             # tile 2 (rows 3..6): channel 2 only
    assert e[2, 0, 0] == 2 and e[2, 1, 1] == (5 - 3) * 4 + 2
