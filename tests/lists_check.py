"""Bit-exact comparison of the CUDA path's paper-level stage-1 lists
(sparse_conv_plane_lists, ISC step 1 of PAPER.md:123) with the oracle's
(oracle.compact_lists): per (image, channel, row tile of TH rows, SURVEY 8c
item 9) the nonzero values with their row and column, row-major, and the
per-list counts.  Test helper (GPU tests and smoke)."""
from __future__ import annotations

import numpy as np

import oracle


def gpu_entries(pl, planes):
    """Flatten a plane_lists() view: (plane, row, col, bits) of every live entry
    in list order, and the exclusive row prefix [planes][H+1]."""
    h, w = pl["h"], pl["w"]
    ent = pl["entries"][:planes].cpu().numpy().view(np.uint32)
    rc = pl["row_counts"][:planes].cpu().numpy().view(np.uint32).astype(np.int64)
    if pl["layout"] == 1:
        tot = rc[:, h]
        live = np.arange(h * w)[None, :] < tot[:, None]
        p, _ = np.nonzero(live)
        bits, pos = ent[live][:, 0], ent[live][:, 1].astype(np.int64)
        prefix = rc
    else:
        live = np.arange(w)[None, None, :] < rc[:, :, None]       # [planes][H][W]
        p, _, _ = np.nonzero(live)
        bits, pos = ent[live][:, 0], ent[live][:, 1].astype(np.int64)
        prefix = np.concatenate([np.zeros((planes, 1), np.int64), np.cumsum(rc, axis=1)], axis=1)
    return p.astype(np.int64), pos // w, pos % w, bits.astype(np.uint32), prefix


def assert_lists_match_oracle(pl, x):
    """pl: SparseConv.plane_lists(n) of a stage 1 run on x (float32 [n][C][H][W],
    host copy of exactly the tensor the GPU read).  Raises AssertionError on the
    first difference."""
    n, c, h, w = x.shape
    planes = n * c
    assert pl["h"] == h and pl["w"] == w
    p, rows, cols, bits, prefix = gpu_entries(pl, planes)
    ref = oracle.compact_lists(x)                                   # TH of SURVEY 8c item 9
    th, tiles = ref["th"], ref["tiles"]
    cnt = ref["counts"].astype(np.int64)                            # [n][C][tiles]
    k = np.arange(ref["values"].shape[-1])
    live = k[None, None, None, :] < cnt[..., None]
    rn, rcn, _, _ = np.nonzero(live)
    r_plane = rn * c + rcn
    assert len(p) == len(r_plane), f"nonzero count {len(p)} != oracle {len(r_plane)}"
    assert np.array_equal(p, r_plane), "entries belong to different planes / order"
    assert np.array_equal(rows, ref["rows"][live]), "row indices differ"
    assert np.array_equal(cols, ref["cols"][live]), "column indices differ"
    assert np.array_equal(bits, ref["values"][live]), "value bits differ"
    # per-list counts at the oracle's row tiling, from the GPU row prefix
    lo = np.minimum(np.arange(tiles) * th, h)
    hi = np.minimum((np.arange(tiles) + 1) * th, h)
    gcnt = (prefix[:, hi] - prefix[:, lo]).reshape(n, c, tiles)
    assert np.array_equal(gcnt, cnt), "per-list counts differ"
    # the row prefix itself against one-row lists
    rows1 = oracle.compact_lists(x, 1)["counts"].astype(np.int64).reshape(planes, h)
    assert np.array_equal(prefix[:, 1:] - prefix[:, :-1], rows1), "row counts differ"
    assert np.all(prefix[:, 0] == 0)


def check_plane_lists(conv, x, n):
    """Paper-level step-1 lists of the plan's last stage 1 (on x[:n]) equal the
    oracle's bit for bit.  Returns False when the plan keeps no plane lists
    (streamwise compaction for planes over 1024 elements / 31 rows)."""
    from paper_1704_07724_b200 import sparseconv as sc
    try:
        pl = conv.plane_lists(n)
    except sc.SparseConvError as e:
        if e.status == 3:
            return False
        raise
    assert_lists_match_oracle(pl, np.ascontiguousarray(x[:n]))
    return True


def check_streams(conv, x, n, ty=None):
    """The kernel's stage-2 streams (R9) equal the test-side adapter's
    derivation from the oracle lists, bit for bit (entries beyond each stream's
    length are never compared).  ty: the tile height the stream layout is
    expected to use (None: the plan's)."""
    import r9_adapter
    p = conv.params
    got = conv.lists(n)
    if ty is not None:
        assert got["ty"] == ty, f"plan tile height {got['ty']} != expected {ty}"
    xs = np.ascontiguousarray(x[:n])
    ref = r9_adapter.streams_from_lists(oracle.compact_lists(xs), xs.shape, p.r, p.stride, p.pad, got["ty"])
    assert (got["tiles"], got["nwr"], got["nwin"], got["cap"]) == (ref["tiles"], ref["nwr"], ref["nwin"], ref["cap"])
    offs = got["offs"].cpu().numpy().view(np.uint32)
    assert np.array_equal(offs, ref["offs"]), "stream offsets differ"
    length = ref["offs"][:, :, -1]
    valid = np.arange(ref["cap"])[None, None, :] < length[:, :, None]
    ge = got["entries"].cpu().numpy().view(np.uint32)
    assert np.array_equal(np.where(valid[..., None], ge, 0), np.where(valid[..., None], ref["entries"], 0)), \
        "stream entries differ"
