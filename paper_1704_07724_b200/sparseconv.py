"""Thin ctypes binding of libsparseconv.so (include/sparse_conv.h).

Argument marshalling only: every step of the convolution runs in the CUDA
kernels of the library.  PyTorch provides device memory and streams.  There
is no CPU fallback: if the library is missing or a call fails, this raises.
"""
from __future__ import annotations

import ctypes
import os

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libsparseconv.so")

SC_FLAG_FUSE_RELU = 1
STATUS = {0: "SC_OK", 1: "SC_ERR_INVALID_ARGUMENT", 2: "SC_ERR_SHAPE", 3: "SC_ERR_UNSUPPORTED",
          4: "SC_ERR_CUDA", 5: "SC_ERR_OUT_OF_MEMORY"}

# every symbol include/sparse_conv.h declares
EXPORTS = ("sparse_conv_output_shape", "sparse_conv_create", "sparse_conv_forward", "dense_conv_forward",
           "sparse_conv_forward_host", "sparse_conv_destroy", "sc_status_string", "sc_last_error",
           "sparse_conv_compact", "sparse_conv_gather", "sparse_conv_lists", "sparse_conv_kernel_variant",
           "sparse_conv_launch_count", "sc_probe_fma", "sc_flush_l2", "sparse_conv_forward_chain",
           "sparse_conv_forward_auto", "sparse_conv_calibrate_crossover", "sparse_conv_set_crossover",
           "sparse_conv_get_crossover", "sparse_conv_last_path", "sparse_conv_backward", "sc_jit_variant_source",
           "sc_jit_available", "sparse_conv_plane_lists", "sparse_conv_forward_batches", "sparse_conv_reserve_batches",
           "sparse_conv_forward_host_batches")
SC_PATH_SPARSE, SC_PATH_DENSE = 0, 1


class SparseConvError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


class ConvParams(ctypes.Structure):
    _fields_ = [(f, ctypes.c_int64) for f in ("n", "c", "h", "w", "k", "r", "s", "stride", "pad", "groups")] + [
        ("flags", ctypes.c_uint32)]


class ListsView(ctypes.Structure):
    _fields_ = [("entries", ctypes.c_void_p), ("offsets", ctypes.c_void_p), ("tiles_per_image", ctypes.c_int64),
                ("stream_capacity", ctypes.c_int64), ("channels", ctypes.c_int64), ("tile_rows", ctypes.c_int32),
                ("window_rows", ctypes.c_int32), ("window_width", ctypes.c_int32), ("marker_code", ctypes.c_int32)]


class PlaneListsView(ctypes.Structure):
    _fields_ = [("entries", ctypes.c_void_p), ("row_counts", ctypes.c_void_p), ("planes", ctypes.c_int64),
                ("height", ctypes.c_int32), ("width", ctypes.c_int32), ("layout", ctypes.c_int32)]


_lib = None


def lib():
    """Load libsparseconv.so.  Raises if it has not been built (no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} is missing: build it with "
                               "`python -c 'import __graft_entry__ as g; g.build()'` (no CPU fallback exists)")
        L = ctypes.CDLL(LIB_PATH)
        vp, i64, st = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int
        L.sparse_conv_output_shape.argtypes = [ctypes.POINTER(ConvParams), ctypes.POINTER(ctypes.c_int64)]
        L.sparse_conv_create.argtypes = [ctypes.POINTER(ConvParams), vp, vp, ctypes.c_int, ctypes.POINTER(vp)]
        for fn in ("sparse_conv_forward", "dense_conv_forward", "sparse_conv_forward_host", "sparse_conv_forward_auto"):
            getattr(L, fn).argtypes = [vp, i64, vp, vp, vp]
        L.sparse_conv_compact.argtypes = [vp, i64, vp, vp]
        L.sparse_conv_forward_chain.argtypes = [ctypes.POINTER(vp), ctypes.c_int32, i64, vp, ctypes.POINTER(vp), vp]
        L.sparse_conv_gather.argtypes = [vp, i64, vp, vp]
        L.sparse_conv_forward_batches.argtypes = [vp, ctypes.c_int32, i64, ctypes.POINTER(vp), ctypes.POINTER(vp), vp]
        L.sparse_conv_reserve_batches.argtypes = [vp]
        L.sparse_conv_forward_host_batches.argtypes = [vp, ctypes.c_int32, i64, ctypes.POINTER(vp), ctypes.POINTER(vp),
                                                       vp]
        L.sparse_conv_destroy.argtypes = [vp]
        L.sparse_conv_lists.argtypes = [vp, ctypes.POINTER(ListsView)]
        L.sparse_conv_kernel_variant.argtypes = [vp, ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(ctypes.c_char_p)]
        L.sparse_conv_launch_count.argtypes = [vp, ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(ctypes.c_int32)]
        L.sparse_conv_backward.argtypes = [vp, i64, vp, vp, vp, vp, vp, vp]
        L.sparse_conv_calibrate_crossover.argtypes = [vp, i64, vp, ctypes.POINTER(ctypes.c_double)]
        L.sparse_conv_set_crossover.argtypes = [vp, ctypes.c_double]
        L.sparse_conv_get_crossover.argtypes = [vp, ctypes.POINTER(ctypes.c_double)]
        L.sparse_conv_last_path.argtypes = [vp, ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(ctypes.c_int64)]
        L.sc_probe_fma.argtypes = [ctypes.c_int32, ctypes.POINTER(ctypes.c_double)]
        L.sc_flush_l2.argtypes = [vp, ctypes.c_size_t, vp]
        L.sc_status_string.argtypes = [st]
        L.sc_status_string.restype = ctypes.c_char_p
        L.sc_last_error.restype = ctypes.c_char_p
        L.sc_jit_variant_source.argtypes = [ctypes.POINTER(ctypes.c_int32), ctypes.c_char_p, ctypes.c_size_t]
        for fn in EXPORTS:
            if fn not in ("sc_status_string", "sc_last_error", "sc_jit_variant_source", "sc_jit_available"):
                getattr(L, fn).restype = st
        L.sc_jit_variant_source.restype = ctypes.c_size_t
        L.sc_jit_available.restype = ctypes.c_int32
        _lib = L
    return _lib


def _check(status):
    if status != 0:
        raise SparseConvError(status, lib().sc_last_error().decode())


def _stream_handle(stream):
    s = torch.cuda.current_stream() if stream is None else stream
    return ctypes.c_void_p(s.cuda_stream)


def _check_tensor(t, name, device, shape=None):
    if not isinstance(t, torch.Tensor) or t.device != device or t.dtype != torch.float32 or not t.is_contiguous():
        raise ValueError(f"{name} must be a contiguous float32 tensor on {device}")
    if shape is not None and tuple(t.shape) != tuple(shape):
        raise ValueError(f"{name} has shape {tuple(t.shape)}, expected {tuple(shape)}")


class _DevArray:
    """__cuda_array_interface__ wrapper so torch can view plan-owned memory."""

    def __init__(self, ptr, shape, typestr):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr, "data": (ptr, False),
                                         "version": 3, "strides": None}


def output_shape(n, c, h, w, k, r, s, stride=1, pad=0, groups=1):
    p = ConvParams(n, c, h, w, k, r, s, stride, pad, groups, 0)
    out = (ctypes.c_int64 * 4)()
    _check(lib().sparse_conv_output_shape(ctypes.byref(p), out))
    return tuple(out)


class SparseConv:
    """One convolution layer: plan-owned packed weights + list workspace.

    weight: [K][C/groups][R][S] float32 CUDA tensor; bias: [K] or None.
    max_batch: the largest n any forward will be called with."""

    def __init__(self, weight, bias, max_batch, c, h, w, stride=1, pad=0, groups=1, fuse_relu=False):
        device = weight.device
        if device.type != "cuda":
            raise ValueError("weight must be a CUDA tensor (there is no CPU path)")
        k, cg, r, s = weight.shape
        _check_tensor(weight, "weight", device)
        if bias is not None:
            _check_tensor(bias, "bias", device, (k,))
        self.device = device
        self.params = ConvParams(max_batch, c, h, w, k, r, s, stride, pad, groups,
                                 SC_FLAG_FUSE_RELU if fuse_relu else 0)
        self.in_shape = (c, h, w)
        self.out_shape = output_shape(max_batch, c, h, w, k, r, s, stride, pad, groups)[1:]
        self._plan = ctypes.c_void_p()
        with torch.cuda.device(device):
            _check(lib().sparse_conv_create(ctypes.byref(self.params), ctypes.c_void_p(weight.data_ptr()),
                                            ctypes.c_void_p(bias.data_ptr()) if bias is not None else None,
                                            device.index if device.index is not None else torch.cuda.current_device(),
                                            ctypes.byref(self._plan)))

    # -- hot path ---------------------------------------------------------
    def forward(self, x, out=None, stream=None):
        n = x.shape[0]
        _check_tensor(x, "x", self.device, (n,) + self.in_shape)
        if out is None:
            out = torch.empty((n,) + self.out_shape, device=self.device, dtype=torch.float32)
        _check_tensor(out, "out", self.device, (n,) + self.out_shape)
        _check(lib().sparse_conv_forward(self._plan, n, ctypes.c_void_p(x.data_ptr()),
                                         ctypes.c_void_p(out.data_ptr()), _stream_handle(stream)))
        return out

    __call__ = forward

    def forward_batches(self, xs, outs=None, stream=None):
        """sparse_conv_forward_batches: independent batches xs[b] -> outs[b] (same batch size),
        batch b+1's stage 1 overlapping batch b's stage 2."""
        n = xs[0].shape[0]
        if outs is None:
            outs = [torch.empty((n,) + self.out_shape, device=self.device, dtype=torch.float32) for _ in xs]
        if len(outs) != len(xs):
            raise ValueError("xs and outs differ in length")
        for x, o in zip(xs, outs):
            _check_tensor(x, "x", self.device, (n,) + self.in_shape)
            _check_tensor(o, "out", self.device, (n,) + self.out_shape)
        ins = (ctypes.c_void_p * len(xs))(*[x.data_ptr() for x in xs])
        ous = (ctypes.c_void_p * len(outs))(*[o.data_ptr() for o in outs])
        _check(lib().sparse_conv_forward_batches(self._plan, len(xs), n, ins, ous, _stream_handle(stream)))
        return outs

    def reserve_batches(self):
        _check(lib().sparse_conv_reserve_batches(self._plan))

    def dense_forward(self, x, out=None, stream=None):
        n = x.shape[0]
        _check_tensor(x, "x", self.device, (n,) + self.in_shape)
        if out is None:
            out = torch.empty((n,) + self.out_shape, device=self.device, dtype=torch.float32)
        _check_tensor(out, "out", self.device, (n,) + self.out_shape)
        _check(lib().dense_conv_forward(self._plan, n, ctypes.c_void_p(x.data_ptr()),
                                        ctypes.c_void_p(out.data_ptr()), _stream_handle(stream)))
        return out

    def forward_auto(self, x, out=None, stream=None):
        """Sparse or dense path, chosen on the device from x's sparsity (f3)."""
        n = x.shape[0]
        _check_tensor(x, "x", self.device, (n,) + self.in_shape)
        if out is None:
            out = torch.empty((n,) + self.out_shape, device=self.device, dtype=torch.float32)
        _check_tensor(out, "out", self.device, (n,) + self.out_shape)
        _check(lib().sparse_conv_forward_auto(self._plan, n, ctypes.c_void_p(x.data_ptr()),
                                              ctypes.c_void_p(out.data_ptr()), _stream_handle(stream)))
        return out

    def calibrate_crossover(self, n, stream=None):
        """Measure the crossover sparsity s* for batches of n; returns it."""
        v = ctypes.c_double()
        with torch.cuda.device(self.device):
            _check(lib().sparse_conv_calibrate_crossover(self._plan, n, _stream_handle(stream), ctypes.byref(v)))
        return v.value

    @property
    def crossover(self):
        """s*: forward_auto takes the sparse path iff the batch sparsity >= s* (None: not set)."""
        v = ctypes.c_double()
        _check(lib().sparse_conv_get_crossover(self._plan, ctypes.byref(v)))
        return None if v.value < 0 else v.value

    @crossover.setter
    def crossover(self, s_star):
        _check(lib().sparse_conv_set_crossover(self._plan, float(s_star)))

    def last_path(self):
        """(path, nnz) of the last forward_auto: path SC_PATH_SPARSE (0) or SC_PATH_DENSE (1)."""
        p, z = ctypes.c_int32(), ctypes.c_int64()
        _check(lib().sparse_conv_last_path(self._plan, ctypes.byref(p), ctypes.byref(z)))
        return p.value, z.value

    def backward(self, x, dout, want_dw=True, want_dbias=True, want_dz=True, stream=None):
        """Gradients of the convolution skipping zero inputs (f4): returns
        (dw [K][C/G][R][S], dbias [K], dz [n][C][H][W]) -- dz is the input
        gradient through the ReLU that produced x (zero where x == 0); an
        output not wanted is None."""
        n = x.shape[0]
        _check_tensor(x, "x", self.device, (n,) + self.in_shape)
        _check_tensor(dout, "dout", self.device, (n,) + self.out_shape)
        p = self.params
        dw = torch.empty((p.k, p.c // p.groups, p.r, p.s), device=self.device) if want_dw else None
        db = torch.empty((p.k,), device=self.device) if want_dbias else None
        dz = torch.empty_like(x) if want_dz else None

        def ptr(t):
            return None if t is None else ctypes.c_void_p(t.data_ptr())

        _check(lib().sparse_conv_backward(self._plan, n, ptr(x), ptr(dout), ptr(dw), ptr(db), ptr(dz),
                                          _stream_handle(stream)))
        return dw, db, dz

    def forward_host(self, h_in, h_out, stream=None):
        """End-to-end call with HOST (ideally pinned) CPU tensors."""
        n = h_in.shape[0]
        for t, nm, shp in ((h_in, "h_in", (n,) + self.in_shape), (h_out, "h_out", (n,) + self.out_shape)):
            if t.device.type != "cpu" or t.dtype != torch.float32 or not t.is_contiguous() or tuple(t.shape) != shp:
                raise ValueError(f"{nm} must be a contiguous float32 CPU tensor of shape {shp}")
        _check(lib().sparse_conv_forward_host(self._plan, n, ctypes.c_void_p(h_in.data_ptr()),
                                              ctypes.c_void_p(h_out.data_ptr()), _stream_handle(stream)))
        return h_out

    def forward_host_batches(self, h_ins, h_outs, stream=None):
        """sparse_conv_forward_host_batches: host batches h_ins[b] -> h_outs[b] (CPU tensors,
        pinned for full bandwidth), copies and kernels of consecutive batches overlapped;
        synchronous."""
        if len(h_ins) != len(h_outs) or not h_ins:
            raise ValueError("h_ins and h_outs must be non-empty and of equal length")
        n = h_ins[0].shape[0]
        for hi, ho in zip(h_ins, h_outs):
            if hi.device.type != "cpu" or ho.device.type != "cpu" or hi.dtype != torch.float32 or \
                    ho.dtype != torch.float32 or not hi.is_contiguous() or not ho.is_contiguous():
                raise ValueError("host batches must be contiguous float32 CPU tensors")
            if tuple(hi.shape) != (n,) + self.in_shape or tuple(ho.shape) != (n,) + self.out_shape:
                raise ValueError("host batch shape mismatch")
        ins = (ctypes.c_void_p * len(h_ins))(*[t.data_ptr() for t in h_ins])
        ous = (ctypes.c_void_p * len(h_outs))(*[t.data_ptr() for t in h_outs])
        _check(lib().sparse_conv_forward_host_batches(self._plan, len(h_ins), n, ins, ous, _stream_handle(stream)))
        return h_outs

    # -- test hooks --------------------------------------------------------
    def compact(self, x, stream=None):
        n = x.shape[0]
        _check_tensor(x, "x", self.device, (n,) + self.in_shape)
        _check(lib().sparse_conv_compact(self._plan, n, ctypes.c_void_p(x.data_ptr()), _stream_handle(stream)))

    def gather(self, n, out=None, stream=None):
        if out is None:
            out = torch.empty((n,) + self.out_shape, device=self.device, dtype=torch.float32)
        _check(lib().sparse_conv_gather(self._plan, n, ctypes.c_void_p(out.data_ptr()), _stream_handle(stream)))
        return out

    def lists(self, n):
        """Device views (int32 bit patterns of the u32 words) of the stage-1
        tile streams of the first n images: dict(entries [n][tiles][cap][2],
        offs [n][tiles][C+1], ty, tiles, nwr, nwin, cap)."""
        v = ListsView()
        _check(lib().sparse_conv_lists(self._plan, ctypes.byref(v)))
        tiles, cap, c = v.tiles_per_image, v.stream_capacity, v.channels
        with torch.cuda.device(self.device):
            entries = torch.as_tensor(_DevArray(v.entries, (n, tiles, cap, 2), "<i4"), device=self.device)
            offs = torch.as_tensor(_DevArray(v.offsets, (n, tiles, c + 1), "<i4"), device=self.device)
        return dict(entries=entries, offs=offs, ty=v.tile_rows, tiles=tiles, nwr=v.window_rows,
                    nwin=v.marker_code, cap=cap)

    def plane_lists(self, n):
        """Device views (int32 bit patterns) of the paper-level stage-1 lists
         of the first n images, as sparse_conv_plane_lists describes:
        dict(layout, entries, row_counts, h, w).  layout 1: entries
        [n*C][H*W][2], row_counts [n*C][H+1] (exclusive row prefix); layout 2:
        entries [n*C][H][W][2] per-row slots, row_counts [n*C][H]."""
        v = PlaneListsView()
        _check(lib().sparse_conv_plane_lists(self._plan, ctypes.byref(v)))
        planes = n * (v.planes // self.params.n)
        h, w = v.height, v.width
        with torch.cuda.device(self.device):
            if v.layout == 1:
                ent = torch.as_tensor(_DevArray(v.entries, (planes, h * w, 2), "<i4"), device=self.device)
                rc = torch.as_tensor(_DevArray(v.row_counts, (planes, h + 1), "<i4"), device=self.device)
            else:
                ent = torch.as_tensor(_DevArray(v.entries, (planes, h, w, 2), "<i4"), device=self.device)
                rc = torch.as_tensor(_DevArray(v.row_counts, (planes, h), "<i4"), device=self.device)
        return dict(layout=v.layout, entries=ent, row_counts=rc, h=h, w=w)

    @property
    def variant(self):
        vid, name = ctypes.c_int32(), ctypes.c_char_p()
        _check(lib().sparse_conv_kernel_variant(self._plan, ctypes.byref(vid), ctypes.byref(name)))
        return vid.value, name.value.decode()

    @property
    def launch_counts(self):
        a, b = ctypes.c_int32(), ctypes.c_int32()
        _check(lib().sparse_conv_launch_count(self._plan, ctypes.byref(a), ctypes.byref(b)))
        return a.value, b.value

    def close(self):
        if self._plan:
            lib().sparse_conv_destroy(self._plan)
            self._plan = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def chain_forward(convs, x, outs, stream=None):
    """Run a chain of SparseConv layers (sparse_conv_forward_chain).  outs[l]:
    output tensor of layer l, or None for an intermediate layer whose epilogue
    should emit the next layer's stage-1 lists instead of a dense output.
    outs[-1] must be a tensor.  Returns outs[-1]."""
    n = x.shape[0]
    _check_tensor(x, "x", convs[0].device, (n,) + convs[0].in_shape)
    for l, (c, o) in enumerate(zip(convs, outs)):
        if o is not None:
            _check_tensor(o, f"outs[{l}]", c.device, (n,) + c.out_shape)
    if outs[-1] is None:
        raise ValueError("the last layer needs an output tensor")
    plans = (ctypes.c_void_p * len(convs))(*[c._plan.value for c in convs])
    ptrs = (ctypes.c_void_p * len(outs))(*[None if o is None else o.data_ptr() for o in outs])
    _check(lib().sparse_conv_forward_chain(plans, len(convs), n, ctypes.c_void_p(x.data_ptr()), ptrs,
                                           _stream_handle(stream)))
    return outs[-1]


def jit_variant_source(R, S, P, T, W, TY, KL, NW=11, MINB=1, CH=16, STAGES=2, SLOTS=3, PIECE=254, vid=1000):
    """Source text of a stage-2 variant generated by the library at run time (test hook)."""
    p = (ctypes.c_int32 * 14)(R, S, P, T, W, TY, KL, NW, MINB, CH, STAGES, SLOTS, PIECE, vid)
    n = lib().sc_jit_variant_source(p, None, 0)
    buf = ctypes.create_string_buffer(n + 1)
    lib().sc_jit_variant_source(p, buf, n + 1)
    return buf.value.decode()


def probe_fma(kind):
    """FP32 pipe probe: lane-FMAs retired per SM clock (kind 0 FFMA, 1 FFMA2, 2 FFMA2+int)."""
    r = ctypes.c_double()
    _check(lib().sc_probe_fma(kind, ctypes.byref(r)))
    return r.value


def flush_l2(scratch, stream=None):
    _check(lib().sc_flush_l2(ctypes.c_void_p(scratch.data_ptr()), scratch.numel() * scratch.element_size(),
                             _stream_handle(stream)))
