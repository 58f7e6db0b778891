"""ctypes binding of libll_b200.so (include/ll.h).  Marshalling only."""

import ctypes
import json
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
lib_path = os.path.join(_HERE, "libll_b200.so")

if not os.path.exists(lib_path):
    raise ImportError(
        "libll_b200.so is not built (%s); run `python paper_2505_23819_b200/build.py` "
        "or __graft_entry__.build() -- there is no fallback path" % lib_path)

_lib = ctypes.CDLL(lib_path)

_c_int64_p = ctypes.POINTER(ctypes.c_int64)
_lib.ll_last_error.restype = ctypes.c_char_p
_lib.ll_version.restype = ctypes.c_char_p
_lib.ll_launch_count.restype = ctypes.c_int64
_lib.ll_layout_create.argtypes = [ctypes.c_int, ctypes.POINTER(ctypes.c_char_p),
                                  ctypes.POINTER(ctypes.c_int), ctypes.c_int,
                                  ctypes.POINTER(ctypes.c_char_p), ctypes.POINTER(ctypes.c_int),
                                  _c_int64_p, ctypes.POINTER(ctypes.c_void_p)]
_lib.ll_layout_destroy.argtypes = [ctypes.c_void_p]
_lib.ll_layout_info.argtypes = [ctypes.c_void_p] + [ctypes.POINTER(ctypes.c_int)] * 4
_lib.ll_layout_get.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.POINTER(ctypes.c_int),
                               ctypes.c_void_p, ctypes.POINTER(ctypes.c_int), _c_int64_p,
                               ctypes.c_size_t]
_lib.ll_compose.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.POINTER(ctypes.c_void_p)]
_lib.ll_invert.argtypes = [ctypes.c_void_p, ctypes.POINTER(ctypes.c_void_p)]
_lib.ll_product.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.POINTER(ctypes.c_void_p)]
_lib.ll_apply.argtypes = [ctypes.c_void_p, _c_int64_p, _c_int64_p]
_lib.ll_layout_props.argtypes = [ctypes.c_void_p] + [ctypes.POINTER(ctypes.c_int)] * 3
_lib.ll_convert.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                            ctypes.c_int, ctypes.c_void_p]


class _Opts(ctypes.Structure):
    _fields_ = [("path", ctypes.c_int), ("batch", ctypes.c_int64), ("max_ctas", ctypes.c_int),
                ("reserved", ctypes.c_int * 8)]


_lib.ll_convert_ex.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                               ctypes.c_void_p, ctypes.c_int, ctypes.POINTER(_Opts),
                               ctypes.c_void_p]
_lib.ll_gather.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                           ctypes.c_int, ctypes.c_int, ctypes.c_void_p]
_lib.ll_gather_ex.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                              ctypes.c_int, ctypes.c_int, ctypes.POINTER(_Opts), ctypes.c_void_p]
_lib.ll_convert_host.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                 ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_void_p,
                                 ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p]
_lib.ll_convert_host_shard.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                       ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                       ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p]
_lib.ll_plan_describe.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_int,
                                  ctypes.c_char_p, ctypes.c_size_t,
                                  ctypes.POINTER(ctypes.c_size_t)]
_lib.ll_gather_describe.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                    ctypes.c_char_p, ctypes.c_size_t,
                                    ctypes.POINTER(ctypes.c_size_t)]
_lib.ll_tune.argtypes = [ctypes.c_char_p, ctypes.c_int]
_VP = ctypes.c_void_p
_lib.ll_mxfp4_upcast.argtypes = [_VP, _VP, _VP, _VP, _VP, _VP, _VP]
_lib.ll_checksum.argtypes = [_VP, ctypes.c_int64, ctypes.c_int, ctypes.c_int, ctypes.c_int64, _VP, _VP]
_lib.ll_transpose.argtypes = [_VP, ctypes.POINTER(ctypes.c_int), ctypes.POINTER(_VP)]
_lib.ll_reshape.argtypes = [_VP, ctypes.c_int, ctypes.POINTER(ctypes.c_char_p),
                            ctypes.POINTER(ctypes.c_int), ctypes.POINTER(_VP)]
_lib.ll_expand_dims.argtypes = [_VP, ctypes.c_int, ctypes.c_char_p, ctypes.POINTER(_VP)]
_lib.ll_broadcast.argtypes = [_VP, ctypes.c_int, ctypes.c_int, ctypes.POINTER(_VP)]
_lib.ll_join.argtypes = [_VP, ctypes.c_char_p, ctypes.POINTER(_VP)]
_lib.ll_split.argtypes = [_VP, ctypes.POINTER(_VP)]
_lib.ll_slice.argtypes = [_VP, ctypes.c_int, ctypes.POINTER(_VP)]
_lib.ll_mxfp4_scale_layout.argtypes = [_VP, ctypes.POINTER(_VP)]
_IP = ctypes.POINTER(ctypes.c_int)
_lib.ll_blocked.argtypes = [ctypes.c_int, _IP, _IP, _IP, _IP, _IP, ctypes.POINTER(_VP)]
_lib.ll_mma_tile.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.POINTER(_VP)]
_lib.ll_convert_shard.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                  ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                  ctypes.c_void_p, ctypes.c_void_p]
_lib.ll_shard_describe.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_int,
                                   ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_int64)]
_lib.ll_gather_host.argtypes = [_VP, _VP, _VP, _VP, ctypes.c_int, ctypes.c_int, ctypes.c_int64,
                                _VP, _VP, _VP, ctypes.c_size_t, _VP]
_lib.ll_shard_describe_2d.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_int,
                                      ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_int64)]
_lib.ll_left_divide.argtypes = [_VP, _VP, ctypes.POINTER(_VP)]
_lib.ll_convert_regs_timed.argtypes = [_VP, _VP, _VP, _VP, ctypes.c_int, ctypes.c_int64,
                                       ctypes.c_int, _VP, _VP]
_lib.ll_convert_inkernel_timed.argtypes = [_VP, _VP, _VP, _VP, ctypes.c_int, ctypes.c_int64,
                                           ctypes.c_int, ctypes.c_int, _VP, _VP]
_lib.ll_jit_source.argtypes = [_VP, _VP, ctypes.c_int, ctypes.c_int, ctypes.c_char_p,
                               ctypes.c_size_t, ctypes.POINTER(ctypes.c_size_t)]
_lib.ll_gather_jit_source.argtypes = [_VP, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                      ctypes.c_char_p, ctypes.c_size_t,
                                      ctypes.POINTER(ctypes.c_size_t)]
_lib.ll_gather_timed.argtypes = [_VP, _VP, _VP, _VP, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                 ctypes.c_int, _VP, _VP]
for _f in ("ll_mxfp4_scale_layout", "ll_slice", "ll_blocked", "ll_mma_tile", "ll_gather_jit_source", "ll_gather_timed", "ll_jit_source", "ll_left_divide", "ll_convert_regs_timed", "ll_convert_inkernel_timed", "ll_mxfp4_upcast", "ll_checksum", "ll_transpose", "ll_reshape", "ll_expand_dims", "ll_broadcast", "ll_join", "ll_split",
           "ll_convert_shard", "ll_shard_describe", "ll_shard_describe_2d", "ll_gather_host", "ll_tune", "ll_layout_create", "ll_layout_destroy", "ll_layout_info", "ll_layout_get",
           "ll_compose", "ll_invert", "ll_product", "ll_apply", "ll_layout_props", "ll_convert",
           "ll_convert_ex", "ll_gather", "ll_gather_ex", "ll_convert_host", "ll_convert_host_shard", "ll_plan_describe",
           "ll_gather_describe"):
    getattr(_lib, _f).restype = ctypes.c_int

STATUS = {0: "LL_OK", 1: "LL_ERR_ARG", 2: "LL_ERR_SHAPE", 3: "LL_ERR_LABEL",
          4: "LL_ERR_NOT_SURJECTIVE", 5: "LL_ERR_NOT_INVERTIBLE", 6: "LL_ERR_RANGE",
          7: "LL_ERR_UNSUPPORTED", 8: "LL_ERR_CUDA", 9: "LL_ERR_OOM"}
PATHS = {"auto": 0, "copy": 1, "smem": 2, "shuffle": 3, "generic": 4, "smem_noswizzle": 5,
         "smem_async": 6, "smem_padded": 7, "smem_tma": 8,
         "regs": 9, "smem_tma_store": 10, "regs_shuffle": 11, "regperm": 12}


class LLError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__("%s: %s" % (STATUS.get(status, status), msg))
        self.status = status
        self.name = STATUS.get(status, str(status))


def _check(st):
    if st != 0:
        raise LLError(st, _lib.ll_last_error().decode())


def version():
    return _lib.ll_version().decode()


def tune(name, value):
    """ll_tune: set a launch-configuration knob (tpg, pipe, gather_vpt)."""
    _check(_lib.ll_tune(name.encode(), int(value)))


def launch_count():
    return int(_lib.ll_launch_count())


class Layout:
    """Owning handle of an ``ll_layout`` (ll_layout_create / ll_layout_destroy)."""

    def __init__(self, in_dims, out_dims, bases, _handle=None):
        if _handle is not None:
            self._h = _handle
            return
        in_dims = [(str(n), int(b)) for n, b in in_dims]
        out_dims = [(str(n), int(b)) for n, b in out_dims]
        n_in, n_out = len(in_dims), len(out_dims)
        in_names = (ctypes.c_char_p * max(1, n_in))(*[n.encode() for n, _ in in_dims])
        in_bits = (ctypes.c_int * max(1, n_in))(*[b for _, b in in_dims])
        out_names = (ctypes.c_char_p * max(1, n_out))(*[n.encode() for n, _ in out_dims])
        out_bits = (ctypes.c_int * max(1, n_out))(*[b for _, b in out_dims])
        flat = []
        for n, b in in_dims:
            vecs = bases.get(n, [])
            if len(vecs) != b:
                raise LLError(1, "dim %s: %d bases given, %d expected" % (n, len(vecs), b))
            for v in vecs:
                if len(v) != n_out:
                    raise LLError(1, "basis arity mismatch")
                flat.extend(int(c) for c in v)
        arr = (ctypes.c_int64 * max(1, len(flat)))(*flat)
        h = ctypes.c_void_p()
        _check(_lib.ll_layout_create(n_in, in_names, in_bits, n_out, out_names, out_bits, arr,
                                     ctypes.byref(h)))
        self._h = h

    @classmethod
    def from_spec(cls, spec):
        return cls(spec["in_dims"], spec["out_dims"], spec["bases"])

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            _lib.ll_layout_destroy(h)
            self._h = None

    @property
    def handle(self):
        return self._h

    def info(self):
        a, b, c, d = (ctypes.c_int() for _ in range(4))
        _check(_lib.ll_layout_info(self._h, ctypes.byref(a), ctypes.byref(b), ctypes.byref(c),
                                   ctypes.byref(d)))
        return a.value, b.value, c.value, d.value

    @property
    def in_bits(self):
        return self.info()[2]

    @property
    def out_bits(self):
        return self.info()[3]

    def spec(self):
        n_in, n_out, tin, _ = self.info()
        in_names = ((ctypes.c_char * 32) * max(1, n_in))()
        out_names = ((ctypes.c_char * 32) * max(1, n_out))()
        in_bits = (ctypes.c_int * max(1, n_in))()
        out_bits = (ctypes.c_int * max(1, n_out))()
        bases = (ctypes.c_int64 * max(1, tin * n_out))()
        _check(_lib.ll_layout_get(self._h, in_names, in_bits, out_names, out_bits, bases,
                                  max(1, tin * n_out)))
        ind = [(in_names[i].value.decode(), in_bits[i]) for i in range(n_in)]
        outd = [(out_names[i].value.decode(), out_bits[i]) for i in range(n_out)]
        res, k = {}, 0
        for n, b in ind:
            res[n] = [tuple(bases[(k + j) * n_out + d] for d in range(n_out)) for j in range(b)]
            k += b
        return {"in_dims": ind, "out_dims": outd, "bases": res}

    def apply(self, coords):
        n_in, n_out, _, _ = self.info()
        ic = (ctypes.c_int64 * max(1, n_in))(*[int(c) for c in coords])
        oc = (ctypes.c_int64 * max(1, n_out))()
        _check(_lib.ll_apply(self._h, ic, oc))
        return tuple(oc[i] for i in range(n_out))

    def props(self):
        a, b, c = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
        _check(_lib.ll_layout_props(self._h, ctypes.byref(a), ctypes.byref(b), ctypes.byref(c)))
        return {"surjective": bool(a.value), "distributed": bool(b.value), "memory": bool(c.value)}


def _wrap(h):
    return Layout(None, None, None, _handle=h)


def compose(outer, inner):
    h = ctypes.c_void_p()
    _check(_lib.ll_compose(outer.handle, inner.handle, ctypes.byref(h)))
    return _wrap(h)


def invert(layout):
    h = ctypes.c_void_p()
    _check(_lib.ll_invert(layout.handle, ctypes.byref(h)))
    return _wrap(h)


def product(a, b):
    h = ctypes.c_void_p()
    _check(_lib.ll_product(a.handle, b.handle, ctypes.byref(h)))
    return _wrap(h)


def left_divide(m, m1):
    """ll_left_divide: m2 with m = [[m1, 0], [0, m2]] label-wise."""
    h = ctypes.c_void_p()
    _check(_lib.ll_left_divide(m.handle, m1.handle, ctypes.byref(h)))
    return _wrap(h)


def transpose(layout, perm):
    """ll_transpose: tt.trans transfer function."""
    h = ctypes.c_void_p()
    p = (ctypes.c_int * max(1, len(perm)))(*[int(x) for x in perm])
    _check(_lib.ll_transpose(layout.handle, p, ctypes.byref(h)))
    return _wrap(h)


def reshape(layout, out_dims):
    """ll_reshape: tt.reshape transfer function; out_dims = [(name, bits)]."""
    h = ctypes.c_void_p()
    n = len(out_dims)
    names = (ctypes.c_char_p * max(1, n))(*[str(a).encode() for a, _ in out_dims])
    bits = (ctypes.c_int * max(1, n))(*[int(b) for _, b in out_dims])
    _check(_lib.ll_reshape(layout.handle, n, names, bits, ctypes.byref(h)))
    return _wrap(h)


def expand_dims(layout, axis, name):
    h = ctypes.c_void_p()
    _check(_lib.ll_expand_dims(layout.handle, int(axis), name.encode(), ctypes.byref(h)))
    return _wrap(h)


def broadcast(layout, axis, bits):
    h = ctypes.c_void_p()
    _check(_lib.ll_broadcast(layout.handle, int(axis), int(bits), ctypes.byref(h)))
    return _wrap(h)


def join(layout, name):
    h = ctypes.c_void_p()
    _check(_lib.ll_join(layout.handle, name.encode(), ctypes.byref(h)))
    return _wrap(h)


def split(layout):
    h = ctypes.c_void_p()
    _check(_lib.ll_split(layout.handle, ctypes.byref(h)))
    return _wrap(h)


def slice_layout(layout, axis):
    """ll_slice: sliced layout, output dim `axis` removed."""
    h = ctypes.c_void_p()
    _check(_lib.ll_slice(layout.handle, int(axis), ctypes.byref(h)))
    return _wrap(h)


def mxfp4_scale_layout(dst_layout):
    """ll_mxfp4_scale_layout: the upcast's scale layout S = (m, kb -> m, kb >> 4)
    o dst_layout (zero columns for kb bits 0-3)."""
    h = ctypes.c_void_p()
    _check(_lib.ll_mxfp4_scale_layout(dst_layout.handle, ctypes.byref(h)))
    return _wrap(h)


def blocked(shape_bits, R, T, W, order):
    """ll_blocked: blocked layout; order[0] = fastest dim."""
    n = len(shape_bits)
    arr = lambda v: (ctypes.c_int * max(1, n))(*[int(x) for x in v])  # noqa: E731
    h = ctypes.c_void_p()
    _check(_lib.ll_blocked(n, arr(shape_bits), arr(R), arr(T), arr(W), arr(order), ctypes.byref(h)))
    return _wrap(h)


def mma_tile(operand, bitwidth):
    """ll_mma_tile: mma.sync fragment tile (reading A8);
    operand "lhs", "rhs" or "out"."""
    op = {"lhs": 0, "rhs": 1, "out": 2}[operand] if isinstance(operand, str) else int(operand)
    h = ctypes.c_void_p()
    _check(_lib.ll_mma_tile(op, int(bitwidth), ctypes.byref(h)))
    return _wrap(h)


def _stream_handle(stream):
    if stream is None:
        import torch
        return torch.cuda.current_stream().cuda_stream
    if isinstance(stream, int):
        return stream
    return stream.cuda_stream


def _ptr(t):
    return t.data_ptr() if hasattr(t, "data_ptr") else int(t)


def _dev_arg(t, name, need_bytes, elem_bits=None):
    """Argument checks for a torch tensor handed to a device entry point (the
    C ABI takes bare pointers, so sizes are checked here): on CUDA,
    contiguous, element width = elem_bits or a raw byte view (uint8), at
    least need_bytes bytes.  Raw integer pointers are passed through unchecked."""
    if not hasattr(t, "data_ptr"):
        return
    if not t.is_cuda:
        raise LLError(1, "%s: tensor is not on a CUDA device" % name)
    if not t.is_contiguous():
        raise LLError(1, "%s: tensor is not contiguous" % name)
    if elem_bits is not None and t.element_size() not in (1, int(elem_bits) // 8):
        raise LLError(1, "%s: element size %d bits != elem_bits %d" % (
            name, t.element_size() * 8, int(elem_bits)))
    have = t.numel() * t.element_size()
    if have < need_bytes:
        raise LLError(1, "%s: %d bytes < %d needed" % (name, have, need_bytes))


def _host_arg(t, name, need_bytes):
    """Argument checks for a host buffer (torch CPU tensor; pinned for full
    speed): on the host, contiguous, at least need_bytes bytes.  Raw integer
    pointers are passed through unchecked."""
    if not hasattr(t, "data_ptr"):
        return
    if getattr(t, "is_cuda", False):
        raise LLError(1, "%s: expected a host (CPU) tensor" % name)
    if not t.is_contiguous():
        raise LLError(1, "%s: tensor is not contiguous" % name)
    have = t.numel() * t.element_size()
    if have < need_bytes:
        raise LLError(1, "%s: %d bytes < %d needed" % (name, have, need_bytes))


def _stream_for(stream, *tensors):
    """The given stream, else the current stream of the first tensor's device."""
    if stream is None:
        for t in tensors:
            if hasattr(t, "device") and getattr(t, "is_cuda", False):
                import torch
                return torch.cuda.current_stream(t.device).cuda_stream
    return _stream_handle(stream)


def _opts(path, batch, max_ctas):
    o = _Opts()
    o.path = PATHS[path] if isinstance(path, str) else int(path)
    o.batch = int(batch)
    o.max_ctas = int(max_ctas)
    return o


def convert(src, A, dst, B, elem_bits, path="auto", batch=1, max_ctas=0, stream=None):
    """ll_convert_ex on device tensors (or raw device pointers as ints)."""
    o = _opts(path, batch, max_ctas)
    wb = int(elem_bits) // 8
    _dev_arg(src, "convert src", (wb << A.in_bits) * int(batch), elem_bits)
    _dev_arg(dst, "convert dst", (wb << B.in_bits) * int(batch), elem_bits)
    _check(_lib.ll_convert_ex(_ptr(src), A.handle, _ptr(dst), B.handle, int(elem_bits),
                              ctypes.byref(o), _stream_for(stream, src, dst)))


def convert_regs_timed(src, A, dst, B, elem_bits, reps=1, cycles=None, batch=1, stream=None,
                       path="regs"):
    """ll_convert_inkernel_timed: register-faithful conversion (path "regs":
    shared memory; "regs_shuffle": warp shuffles, A -> B -> A per rep), the
    exchange repeated `reps` times in-kernel; per-CTA clock64 cycles into
    `cycles` (an int64 device tensor) when given."""
    _check(_lib.ll_convert_inkernel_timed(_ptr(src), A.handle, _ptr(dst), B.handle,
                                          int(elem_bits), int(batch),
                                          PATHS[path] if isinstance(path, str) else int(path),
                                          int(reps), _ptr(cycles) if cycles is not None else None,
                                          _stream_handle(stream)))


def jit_source(A, B, elem_bits, compile=False, kernel="regs_shuffle"):
    """ll_jit_source: the NVRTC-specialised kernel source (kernel
    "regs_shuffle" or "shuffle" = the HBM shuffle conversion, "smem",
    "upcast", "regperm", "tma" / "tma_store" = the warp-specialised TMA
    kernels), or with
    compile=True the NVRTC compile result as a dict."""
    mode = (1 if compile else 0) | (2 if kernel == "shuffle" else 0) | (4 if kernel == "smem" else 0) \
        | (8 if kernel == "upcast" else 0) | (16 if kernel == "regperm" else 0) \
        | (32 if kernel == "tma" else 0) | (64 if kernel == "tma_store" else 0)
    need = ctypes.c_size_t()
    _check(_lib.ll_jit_source(A.handle, B.handle, int(elem_bits), mode, None, 0,
                              ctypes.byref(need)))
    buf = ctypes.create_string_buffer(need.value)
    _check(_lib.ll_jit_source(A.handle, B.handle, int(elem_bits), mode, buf, need.value,
                              ctypes.byref(need)))
    out = buf.value.decode()
    return json.loads(out) if compile else out


def convert_shard(src_slice, A, dst_slice, B, elem_bits, n_shards, shard, path="auto",
                  max_ctas=0, stream=None):
    """ll_convert_shard: convert this rank's slice."""
    o = _opts(path, 1, max_ctas)
    wb = int(elem_bits) // 8
    if int(n_shards) >= 1:
        _dev_arg(src_slice, "convert_shard src", (wb << A.in_bits) // int(n_shards), elem_bits)
        _dev_arg(dst_slice, "convert_shard dst", (wb << B.in_bits) // int(n_shards), elem_bits)
    _check(_lib.ll_convert_shard(_ptr(src_slice), A.handle, _ptr(dst_slice), B.handle,
                                 int(elem_bits), int(n_shards), int(shard), ctypes.byref(o),
                                 _stream_for(stream, src_slice, dst_slice)))


def mxfp4_upcast(packed, A, scales, dst_bf16, B, max_ctas=0, stream=None):
    """ll_mxfp4_upcast: packed E2M1 bytes (layout A) + E8M0 scales [M][K/32]
    -> bf16, two per byte of B (fused with the conversion)."""
    o = _opts("auto", 1, max_ctas)
    _dev_arg(packed, "mxfp4_upcast packed", 1 << A.in_bits)
    _dev_arg(scales, "mxfp4_upcast scales", (1 << A.in_bits) // 16)
    _dev_arg(dst_bf16, "mxfp4_upcast dst_bf16", 4 << B.in_bits)
    _check(_lib.ll_mxfp4_upcast(_ptr(packed), A.handle, _ptr(scales), _ptr(dst_bf16), B.handle,
                                ctypes.byref(o), _stream_for(stream, packed, dst_bf16)))


def checksum(buf, n_elems, elem_bits, result, indexed=True, index_base=0, stream=None):
    """ll_checksum into the device uint64 `result` (a 1-element int64 tensor or
    a device pointer); enqueued on `stream`, no synchronisation."""
    _dev_arg(buf, "checksum buf", int(n_elems) * int(elem_bits) // 8)
    _dev_arg(result, "checksum result", 8)
    _check(_lib.ll_checksum(_ptr(buf), int(n_elems), int(elem_bits), 1 if indexed else 0,
                            int(index_base), _ptr(result), _stream_handle(stream)))


def shard_describe(A, B, elem_bits, n_shards, shard, path="auto"):
    """Byte ranges (src_begin, src_end, dst_begin, dst_end) of one shard."""
    out = (ctypes.c_int64 * 4)()
    _check(_lib.ll_shard_describe(A.handle, B.handle, int(elem_bits),
                                  PATHS[path] if isinstance(path, str) else int(path),
                                  int(n_shards), int(shard), out))
    return tuple(out)


def gather_host(src_host, idx_host, out_host, L, axis, elem_bits, batch, dev_src, dev_idx,
                dev_out, scratch_bytes, stream=None):
    """ll_gather_host: host buffers in, host buffer out (pipelined copies)."""
    wb, n = int(elem_bits) // 8, (1 << L.in_bits) * int(batch)
    _host_arg(src_host, "gather_host src_host", wb * n)
    _host_arg(idx_host, "gather_host idx_host", 4 * n)
    _host_arg(out_host, "gather_host out_host", wb * n)
    for t, nm in ((dev_src, "dev_src"), (dev_idx, "dev_idx"), (dev_out, "dev_out")):
        _dev_arg(t, "gather_host " + nm, int(scratch_bytes))
    _check(_lib.ll_gather_host(_ptr(src_host), _ptr(idx_host), _ptr(out_host), L.handle, int(axis),
                               int(elem_bits), int(batch), _ptr(dev_src), _ptr(dev_idx),
                               _ptr(dev_out), int(scratch_bytes), _stream_handle(stream)))


def shard_describe_2d(A, B, elem_bits, n_shards, shard, path="auto"):
    """Pitched shard: (side, r0, contiguous begin, end, row bytes, pitch)."""
    out = (ctypes.c_int64 * 6)()
    _check(_lib.ll_shard_describe_2d(A.handle, B.handle, int(elem_bits),
                                     PATHS[path] if isinstance(path, str) else int(path),
                                     int(n_shards), int(shard), out))
    return tuple(out)


def gather(src, idx, out, L, axis, elem_bits, path="auto", batch=1, max_ctas=0, stream=None):
    o = _opts(path, batch, max_ctas)
    n = (1 << L.in_bits) * int(batch)
    _dev_arg(src, "gather src", n * (int(elem_bits) // 8), elem_bits)
    _dev_arg(idx, "gather idx", n * 4, 32)
    _dev_arg(out, "gather out", n * (int(elem_bits) // 8), elem_bits)
    _check(_lib.ll_gather_ex(_ptr(src), _ptr(idx), _ptr(out), L.handle, int(axis),
                             int(elem_bits), ctypes.byref(o), _stream_for(stream, src, idx, out)))


def convert_host(src_host, A, dst_host, B, elem_bits, batch, dev_src, dev_dst, scratch_bytes,
                 stream=None):
    """ll_convert_host: host buffers in, host buffers out (pipelined copies)."""
    wb, nb = int(elem_bits) // 8, max(1, int(batch))
    _host_arg(src_host, "convert_host src_host", (wb << A.in_bits) * nb)
    _host_arg(dst_host, "convert_host dst_host", (wb << B.in_bits) * nb)
    _dev_arg(dev_src, "convert_host dev_src", int(scratch_bytes))
    _dev_arg(dev_dst, "convert_host dev_dst", int(scratch_bytes))
    _check(_lib.ll_convert_host(_ptr(src_host), A.handle, _ptr(dst_host), B.handle,
                                int(elem_bits), int(batch), _ptr(dev_src), _ptr(dev_dst),
                                int(scratch_bytes), _stream_handle(stream)))


def convert_host_shard(src_host, A, dst_host, B, elem_bits, n_shards, shard, dev_src, dev_dst,
                       scratch_bytes, stream=None):
    """ll_convert_host_shard: one rank's shard from host slices (pipelined)."""
    wb, ns = int(elem_bits) // 8, max(1, int(n_shards))
    _host_arg(src_host, "convert_host_shard src_host", (wb << A.in_bits) // ns)
    _host_arg(dst_host, "convert_host_shard dst_host", (wb << B.in_bits) // ns)
    _dev_arg(dev_src, "convert_host_shard dev_src", int(scratch_bytes))
    _dev_arg(dev_dst, "convert_host_shard dev_dst", int(scratch_bytes))
    _check(_lib.ll_convert_host_shard(_ptr(src_host), A.handle, _ptr(dst_host), B.handle,
                                      int(elem_bits), int(n_shards), int(shard), _ptr(dev_src),
                                      _ptr(dev_dst), int(scratch_bytes), _stream_handle(stream)))


def _describe(fn, *args):
    need = ctypes.c_size_t()
    _check(fn(*args, None, 0, ctypes.byref(need)))
    buf = ctypes.create_string_buffer(need.value + 1)
    _check(fn(*args, buf, need.value + 1, ctypes.byref(need)))
    return json.loads(buf.value.decode())


def plan_describe(A, B, elem_bits, path="auto"):
    return _describe(_lib.ll_plan_describe, A.handle, B.handle, int(elem_bits),
                     PATHS[path] if isinstance(path, str) else int(path))


def gather_describe(L, axis, elem_bits, path="auto"):
    return _describe(_lib.ll_gather_describe, L.handle, int(axis), int(elem_bits),
                     PATHS[path] if isinstance(path, str) else int(path))


def gather_jit_source(L, axis, elem_bits, path="shuffle", compile=False, timed=False):
    """ll_gather_jit_source: the compiled gather kernel's CUDA source (or,
    compile=True, the NVRTC result as a dict)."""
    mode = (1 if compile else 0) | (2 if timed else 0)
    p = PATHS[path] if isinstance(path, str) else int(path)
    need = ctypes.c_size_t()
    _check(_lib.ll_gather_jit_source(L.handle, int(axis), int(elem_bits), p, mode, None, 0,
                                     ctypes.byref(need)))
    buf = ctypes.create_string_buffer(need.value)
    _check(_lib.ll_gather_jit_source(L.handle, int(axis), int(elem_bits), p, mode, buf,
                                     need.value, ctypes.byref(need)))
    out = buf.value.decode()
    return json.loads(out) if compile else out


def gather_timed(src, idx, out, L, axis, elem_bits, path, reps, cycles, stream=None):
    """ll_gather_timed: one CTA, the gather exchange repeated `reps` times
    in-kernel; clock64 cycles into cycles[0] (int64 device tensor)."""
    _check(_lib.ll_gather_timed(_ptr(src), _ptr(idx), _ptr(out), L.handle, int(axis),
                                int(elem_bits), PATHS[path] if isinstance(path, str) else int(path),
                                int(reps), _ptr(cycles), _stream_for(stream, src, idx, out)))
