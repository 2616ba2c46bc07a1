"""Thin ctypes binding of ``include/lic.h`` (argument marshalling only).

Every step of the codec runs in ``liblic.so`` (sm_100a kernels + the native host coder);
there is no Python or CPU fallback: if the library is missing this module raises on
import.  Arrays may be numpy arrays (host memory) or torch tensors (device or pinned
host memory); they are passed to the C ABI as raw pointers.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# LIC_LIB: an alternative in-tree build of the same library (A/B experiments, scripts/ab_lib.sh)
LIB_PATH = os.path.join(_HERE, os.environ.get("LIC_LIB", "liblic.so"))

LIC_OK, LIC_EINVAL, LIC_ESHAPE, LIC_ECORRUPT, LIC_EDIGEST, LIC_ENOMEM, LIC_ECUDA, LIC_EFOREIGN, \
    LIC_ENOSPACE = range(9)
PREC_SPLIT, PREC_F16 = 0, 1
LAYERS = ["ga1", "ga2", "ga3", "ga4", "gs1", "gs2", "gs3", "gs4", "ha1", "ha2", "ha3", "hs1", "hs2", "hs3"]


class LicError(RuntimeError):
    def __init__(self, status, msg=""):
        super().__init__(f"lic status {status}: {msg}")
        self.status = status


class CorruptStream(LicError):
    pass


class Shape(ctypes.Structure):
    _fields_ = [("c", ctypes.c_uint32), ("h", ctypes.c_uint32), ("w", ctypes.c_uint32)]

    def tuple(self):
        return (self.c, self.h, self.w)


if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is not built: run `python -m paper_2208_01641_b200.build` "
                      "(there is no fallback path)")
_L = ctypes.CDLL(LIB_PATH)
_P = ctypes.c_void_p
_u32, _sz, _i = ctypes.c_uint32, ctypes.c_size_t, ctypes.c_int
_L.lic_open.argtypes = [_P, _sz, _i, _u32, _u32, _u32, _i, ctypes.POINTER(_P)]
_L.lic_close.argtypes = [_P]
_L.lic_close.restype = None
_L.lic_shapes.argtypes = [_P, ctypes.POINTER(Shape), ctypes.POINTER(Shape), ctypes.POINTER(_i)]
_L.lic_last_error.argtypes = [_P]
_L.lic_last_error.restype = ctypes.c_char_p
_L.lic_buf_acquire.argtypes = [_P, _sz, ctypes.POINTER(_P)]
_L.lic_buf_release.argtypes = [_P, _P]
_L.lic_buf_stats.argtypes = [_P, ctypes.POINTER(ctypes.c_uint64), ctypes.POINTER(ctypes.c_uint64)]
_L.lic_encode.argtypes = [_P, _P, _u32, _P, _P, _P, _P, _P]
_L.lic_encode_u8.argtypes = [_P, _P, _u32, _P, _P, _P, _P, _P]
_L.lic_hyper_indexes.argtypes = [_P, _P, _u32, _P, _P]
_L.lic_decode.argtypes = [_P, _P, _u32, _P, _P]
_L.lic_decode_u8.argtypes = [_P, _P, _u32, _P, _P]
_L.lic_test_layer.argtypes = [_P, _i, _P, _u32, _P, _P]
_L.lic_layer_shapes.argtypes = [_P, _i, ctypes.POINTER(Shape), ctypes.POINTER(Shape)]
_L.lic_test_sigma_to_index.argtypes = [_P, _P, _sz, _P]
_L.lic_set_debug.argtypes = [_P, _i]
_L.lic_debug_latents.argtypes = [_P, _u32, _P, _P, _P]
_L.lic_cdf.argtypes = [_P, _i, ctypes.POINTER(ctypes.POINTER(ctypes.c_uint32)), ctypes.POINTER(_u32),
                       ctypes.POINTER(_u32)]
_L.lic_cdf_build.argtypes = [_P, _u32, _u32, _P]
_L.lic_rans_encode.argtypes = [_P, _P, Shape, _P, _u32, _u32, _i, _P, _sz, ctypes.POINTER(_sz)]
_L.lic_rans_decode.argtypes = [_P, _sz, _P, Shape, _P, _u32, _u32, _i, _P]
_L.lic_version.restype = ctypes.c_char_p
_L.lic_profile.argtypes = [_P, _i]
_L.lic_profile_layers.argtypes = [_P, _u32]
_L.lic_profile_read.argtypes = [_P, _i, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_uint64)]
_L.lic_launch_count.argtypes = [_P, ctypes.POINTER(ctypes.c_uint64)]
_L.lic_set_zero_copy.argtypes = [_P, _i]
_L.lic_trace.argtypes = [_P, _i, _i]
_L.lic_trace_read.argtypes = [_P, _P, _sz]
_L.lic_workspace_bytes.argtypes = [_P, _u32]
_L.lic_workspace_bytes.restype = _sz
_L.lic_bind_workspace.argtypes = [_P, _P, _sz]
_L.lic_max_batch.argtypes = [_P, ctypes.POINTER(_u32)]
_L.lic_range_count.argtypes = [_P, ctypes.POINTER(ctypes.c_uint64), _i]



class PipelineConfig(ctypes.Structure):
    _fields_ = [("coder_threads", ctypes.c_uint32), ("batch", ctypes.c_uint32), ("inflight", ctypes.c_uint32),
                ("u8", ctypes.c_int), ("serial", ctypes.c_int), ("keep_bitstreams", ctypes.c_int),
                ("substreams", ctypes.c_uint32), ("coder", ctypes.c_uint32), ("pace_fps", ctypes.c_float),
                ("timeline", ctypes.c_uint32), ("coder_parts", ctypes.c_uint32)]


class TimelineEvent(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_uint32), ("lane", ctypes.c_uint32), ("batch", ctypes.c_int32),
                ("frame", ctypes.c_int32), ("t_ready_ms", ctypes.c_double), ("t_start_ms", ctypes.c_double),
                ("t_end_ms", ctypes.c_double)]


TIMELINE_KINDS = ["gpu_encode", "gpu_hyper_indexes", "gpu_decode", "coder_enc+dec_z", "coder_dec_y"]


class PipelineStats(ctypes.Structure):
    _fields_ = [("frames", ctypes.c_uint64), ("seconds", ctypes.c_double), ("latency_p50_ms", ctypes.c_double),
                ("latency_p95_ms", ctypes.c_double), ("latency_max_ms", ctypes.c_double),
                ("y_bytes", ctypes.c_uint64), ("z_bytes", ctypes.c_uint64), ("symbol_mismatches", ctypes.c_uint64),
                ("gpu_busy_s", ctypes.c_double), ("coder_busy_s", ctypes.c_double),
                ("gpu_launches", ctypes.c_uint64)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


_L.lic_pipeline_open.argtypes = [_P, ctypes.POINTER(PipelineConfig), ctypes.POINTER(_P)]
_L.lic_pipeline_close.argtypes = [_P]
_L.lic_pipeline_close.restype = None
_L.lic_pipeline_run.argtypes = [_P, _P, _u32, _P, ctypes.POINTER(PipelineStats)]
_L.lic_pipeline_timeline.argtypes = [_P, ctypes.POINTER(TimelineEvent), _sz, ctypes.POINTER(_sz)]
_L.lic_pipeline_bitstream.argtypes = [_P, _u32, ctypes.POINTER(ctypes.POINTER(ctypes.c_uint8)),
                                      ctypes.POINTER(_sz), ctypes.POINTER(ctypes.POINTER(ctypes.c_uint8)),
                                      ctypes.POINTER(_sz)]

_L.lic_rans_prepare.argtypes = [_P, _u32, _u32, _i, ctypes.POINTER(_P)]
_L.lic_rans_tables_free.argtypes = [_P]
_L.lic_rans_tables_free.restype = None
_L.lic_rans_encode_fast.argtypes = [_P, _P, _P, Shape, _P, _sz, ctypes.POINTER(_sz)]
_L.lic_rans_decode_fast.argtypes = [_P, _P, _sz, _P, Shape, _P]
_L.lic_rans_encode_slabs.argtypes = [_P, _P, _P, Shape, _u32, _P, _sz, ctypes.POINTER(_sz)]
_L.lic_rans_decode_slabs.argtypes = [_P, _P, _sz, _P, Shape, _u32, _P]
_L.lic_rans_encode_slab_range.argtypes = [_P, _P, _P, Shape, _u32, _u32, _u32, _P, _sz, _P, ctypes.POINTER(_sz)]
_L.lic_rans_decode_slab_range.argtypes = [_P, _P, _sz, _P, Shape, _u32, _u32, _u32, _P]
_L.lic_cdf_quantize.argtypes = [_P, _u32, _P]
_L.lic_sigmas.argtypes = [_P, _i, ctypes.POINTER(ctypes.POINTER(ctypes.c_float)), ctypes.POINTER(_u32)]
_L.lic_cdf64_gaussian.argtypes = [_P, _u32, ctypes.c_double, _P, _u32, _P, _P]
_L.lic_rans64_encode.argtypes = [_P, _P, _sz, _P, _u32, _u32, _P, _P, _P, _sz, ctypes.POINTER(_sz)]
_L.lic_rans64_decode.argtypes = [_P, _sz, _P, _sz, _P, _u32, _u32, _P, _P, _P]

EXPORTED = [n for n in dir(_L) if n.startswith("lic_")]


def lib():
    return _L


def _ptr(a):
    """Raw address of a numpy array / torch tensor / int / None."""
    if a is None:
        return None
    if isinstance(a, int):
        return a
    if isinstance(a, np.ndarray):
        if not a.flags["C_CONTIGUOUS"]:
            raise ValueError("array must be C-contiguous")
        return a.ctypes.data
    if hasattr(a, "data_ptr"):
        if not a.is_contiguous():
            raise ValueError("tensor must be contiguous")
        return a.data_ptr()
    raise TypeError(type(a))


def _stream(s):
    if s is None:
        return None
    return s.cuda_stream if hasattr(s, "cuda_stream") else int(s)


def version():
    return _L.lic_version().decode()


# ---------------------------------------------------------------- host coder
def cdf_build(sigmas, L):
    s = np.ascontiguousarray(sigmas, np.float32)
    out = np.empty((s.size, 2 * L + 2), np.uint32)
    st = _L.lic_cdf_build(_ptr(s), s.size, L, _ptr(out))
    if st:
        raise LicError(st, "cdf_build")
    return out


def rans_encode(sym, cdf, rows=None, sym_min=None):
    """sym: int8 [C,H,W] (rows None -> row = channel) or any shape with uint8 rows."""
    sym = np.ascontiguousarray(sym, np.int8)
    cdf = np.ascontiguousarray(cdf, np.uint32)
    if sym.ndim == 3:
        shp = Shape(*sym.shape)
    else:
        shp = Shape(1, 1, sym.size)
    if rows is not None:
        rows = np.ascontiguousarray(rows, np.uint8)
        assert rows.size == sym.size
    if sym_min is None:
        sym_min = -((cdf.shape[1] - 2) // 2)
    cap = 2 * sym.size + 64
    out = np.empty(cap, np.uint8)
    n = ctypes.c_size_t(0)
    st = _L.lic_rans_encode(_ptr(sym), _ptr(rows), shp, _ptr(cdf), cdf.shape[0], cdf.shape[1], int(sym_min),
                            _ptr(out), cap, ctypes.byref(n))
    if st:
        raise LicError(st, "rans_encode")
    return out[: n.value].tobytes()


def rans_decode(data, shape, cdf, rows=None, sym_min=None, out=None):
    cdf = np.ascontiguousarray(cdf, np.uint32)
    shp = Shape(*shape) if len(shape) == 3 else Shape(1, 1, int(np.prod(shape)))
    if rows is not None:
        rows = np.ascontiguousarray(rows, np.uint8)
    if sym_min is None:
        sym_min = -((cdf.shape[1] - 2) // 2)
    if out is None:
        out = np.empty(shape, np.int8)
    buf = np.frombuffer(bytes(data), np.uint8) if len(data) else np.zeros(1, np.uint8)
    st = _L.lic_rans_decode(_ptr(buf), len(data), _ptr(rows), shp, _ptr(cdf), cdf.shape[0], cdf.shape[1],
                            int(sym_min), _ptr(out))
    if st == LIC_ECORRUPT:
        raise CorruptStream(st, "corrupt stream")
    if st:
        raise LicError(st, "rans_decode")
    return out


def cdf_quantize(pmf):
    """lic_cdf_quantize: quantised CDF (len(pmf) + 1 entries) of a pmf whose last entry is
    the escape's tail mass."""
    p = np.ascontiguousarray(pmf, np.float32)
    out = np.empty(p.size + 1, np.uint32)
    st = _L.lic_cdf_quantize(_ptr(p), p.size, _ptr(out))
    if st:
        raise LicError(st, "cdf_quantize")
    return out


class Rans64Tables:
    """Tables of the rans64 + bypass coder (lic_rans64_*, R23): cdfs [n, stride]
    uint32, sizes [n] int32, offsets [n] int32."""

    def __init__(self, cdfs, sizes, offsets):
        self.cdfs = np.ascontiguousarray(cdfs, np.uint32)
        self.sizes = np.ascontiguousarray(sizes, np.int32)
        self.offsets = np.ascontiguousarray(offsets, np.int32)
        assert self.cdfs.ndim == 2 and self.sizes.shape == self.offsets.shape == (self.cdfs.shape[0],)

    @classmethod
    def gaussian(cls, scales, tail_mass=1e-9, stride=None):
        """lic_cdf64_gaussian: one row per scale (CompressAI's GaussianConditional tables)."""
        s = np.ascontiguousarray(scales, np.float32)
        if stride is None:
            stride = 2 * int(np.ceil(float(s.max()) * 6.2)) + 8
        cdfs = np.zeros((s.size, stride), np.uint32)
        sizes = np.zeros(s.size, np.int32)
        offs = np.zeros(s.size, np.int32)
        st = _L.lic_cdf64_gaussian(_ptr(s), s.size, float(tail_mass), _ptr(cdfs), stride, _ptr(sizes), _ptr(offs))
        if st:
            raise LicError(st, "cdf64_gaussian")
        return cls(cdfs, sizes, offs)

    def encode(self, sym, idx):
        sym = np.ascontiguousarray(sym, np.int32).ravel()
        idx = np.ascontiguousarray(idx, np.int32).ravel()
        if sym.size != idx.size:
            raise ValueError("sym / idx sizes differ")
        cap = 8 + 8 * sym.size
        out = np.empty(cap, np.uint8)
        n = _sz(0)
        st = _L.lic_rans64_encode(_ptr(sym), _ptr(idx), sym.size, _ptr(self.cdfs), self.cdfs.shape[0],
                                  self.cdfs.shape[1], _ptr(self.sizes), _ptr(self.offsets), _ptr(out), cap,
                                  ctypes.byref(n))
        if st:
            raise LicError(st, "rans64_encode")
        return out[: n.value].tobytes()

    def decode(self, data, idx):
        idx = np.ascontiguousarray(idx, np.int32).ravel()
        buf = np.frombuffer(bytes(data), np.uint8) if len(data) else np.zeros(1, np.uint8)
        out = np.empty(idx.size, np.int32)
        st = _L.lic_rans64_decode(_ptr(buf), len(data), _ptr(idx), idx.size, _ptr(self.cdfs), self.cdfs.shape[0],
                                  self.cdfs.shape[1], _ptr(self.sizes), _ptr(self.offsets), _ptr(out))
        if st == LIC_ECORRUPT:
            raise CorruptStream(st, "rans64_decode")
        if st:
            raise LicError(st, "rans64_decode")
        return out


class RansTables:
    """lic_rans_prepare: prepared (fast) coder tables, same bitstream as rans_encode."""

    def __init__(self, cdf, sym_min=None):
        self.cdf = np.ascontiguousarray(cdf, np.uint32)
        if sym_min is None:
            sym_min = -((self.cdf.shape[1] - 2) // 2)
        self._h = _P()
        st = _L.lic_rans_prepare(_ptr(self.cdf), self.cdf.shape[0], self.cdf.shape[1], int(sym_min),
                                 ctypes.byref(self._h))
        if st:
            raise LicError(st, "lic_rans_prepare")

    def encode(self, sym, rows=None, substreams=1):
        """lic_rans_encode_fast (substreams = 1) or lic_rans_encode_slabs (K channel slabs)."""
        sym = np.ascontiguousarray(sym, np.int8)
        shp = Shape(*sym.shape) if sym.ndim == 3 else Shape(1, 1, sym.size)
        rows = None if rows is None else np.ascontiguousarray(rows, np.uint8)
        cap = 2 * sym.size + 64 + 8 * substreams
        out = np.empty(cap, np.uint8)
        n = ctypes.c_size_t(0)
        if substreams == 1:
            st = _L.lic_rans_encode_fast(self._h, _ptr(sym), _ptr(rows), shp, _ptr(out), cap, ctypes.byref(n))
        else:
            st = _L.lic_rans_encode_slabs(self._h, _ptr(sym), _ptr(rows), shp, substreams, _ptr(out), cap,
                                          ctypes.byref(n))
        if st:
            raise LicError(st, "rans_encode_fast")
        return out[: n.value].tobytes()

    def encode_range(self, sym, K, k_begin, k_end, rows=None):
        """lic_rans_encode_slab_range: (strings of slabs [k_begin, k_end) back to back, their lengths)."""
        sym = np.ascontiguousarray(sym, np.int8)
        rows = None if rows is None else np.ascontiguousarray(rows, np.uint8)
        cap = 2 * sym.size + 64 * K
        out = np.empty(cap, np.uint8)
        lens = np.zeros(k_end - k_begin, np.uint32)
        n = ctypes.c_size_t(0)
        st = _L.lic_rans_encode_slab_range(self._h, _ptr(sym), _ptr(rows), Shape(*sym.shape), K, k_begin, k_end,
                                           _ptr(out), cap, _ptr(lens), ctypes.byref(n))
        if st:
            raise LicError(st, "rans_encode_slab_range")
        return out[: n.value].tobytes(), lens

    def decode_range(self, data, shape, K, k_begin, k_end, rows=None, out=None):
        """lic_rans_decode_slab_range: slabs [k_begin, k_end) of the framed stream into `out`."""
        rows = None if rows is None else np.ascontiguousarray(rows, np.uint8)
        out = np.zeros(shape, np.int8) if out is None else out
        buf = np.frombuffer(bytes(data), np.uint8) if len(data) else np.zeros(1, np.uint8)
        st = _L.lic_rans_decode_slab_range(self._h, _ptr(buf), len(data), _ptr(rows), Shape(*shape), K, k_begin, k_end,
                                           _ptr(out))
        if st == LIC_ECORRUPT:
            raise CorruptStream(st, "corrupt stream")
        if st:
            raise LicError(st, "rans_decode_slab_range")
        return out

    def decode(self, data, shape, rows=None, substreams=1):
        shp = Shape(*shape) if len(shape) == 3 else Shape(1, 1, int(np.prod(shape)))
        rows = None if rows is None else np.ascontiguousarray(rows, np.uint8)
        out = np.empty(shape, np.int8)
        buf = np.frombuffer(bytes(data), np.uint8) if len(data) else np.zeros(1, np.uint8)
        if substreams == 1:
            st = _L.lic_rans_decode_fast(self._h, _ptr(buf), len(data), _ptr(rows), shp, _ptr(out))
        else:
            st = _L.lic_rans_decode_slabs(self._h, _ptr(buf), len(data), _ptr(rows), shp, substreams, _ptr(out))
        if st == LIC_ECORRUPT:
            raise CorruptStream(st, "corrupt stream")
        if st:
            raise LicError(st, "rans_decode_fast")
        return out

    def __del__(self):
        try:
            _L.lic_rans_tables_free(self._h)
        except Exception:
            pass


# ---------------------------------------------------------------- codec
class Codec:
    """One lic_codec: (weights, geometry, device, max_batch)."""

    def __init__(self, licw: bytes, height: int, width: int, max_batch: int = 1, device: int = 0,
                 precision: int = PREC_SPLIT):
        self._h = _P()
        buf = (ctypes.c_uint8 * len(licw)).from_buffer_copy(licw)
        st = _L.lic_open(buf, len(licw), device, height, width, max_batch, precision, ctypes.byref(self._h))
        if st:
            msg = _L.lic_last_error(None)
            raise LicError(st, "lic_open" + (f": {msg.decode()}" if msg else ""))
        self.height, self.width, self.max_batch = height, width, max_batch
        y, z, k = Shape(), Shape(), _i()
        _L.lic_shapes(self._h, ctypes.byref(y), ctypes.byref(z), ctypes.byref(k))
        self.y_shape, self.z_shape, self.hyper = y.tuple(), z.tuple(), bool(k.value)

    def close(self):
        if self._h:
            _L.lic_close(self._h)
            self._h = _P()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _chk(self, st, what):
        if st:
            msg = _L.lic_last_error(self._h)
            raise LicError(st, f"{what}: {msg.decode() if msg else ''}")

    @property
    def handle(self):
        return self._h

    # -- tables
    def sigmas(self, which):
        """lic_sigmas: 0 sigma_y (factorized), 1 sigma_z, 2 the scale table (hyperprior)."""
        ptr = ctypes.POINTER(ctypes.c_float)()
        n = _u32()
        self._chk(_L.lic_sigmas(self._h, which, ctypes.byref(ptr), ctypes.byref(n)), "lic_sigmas")
        return np.ctypeslib.as_array(ptr, shape=(n.value,)).copy()

    def cdf(self, which):
        rows = ctypes.POINTER(ctypes.c_uint32)()
        n, rl = _u32(), _u32()
        self._chk(_L.lic_cdf(self._h, which, ctypes.byref(rows), ctypes.byref(n), ctypes.byref(rl)), "lic_cdf")
        return np.ctypeslib.as_array(rows, shape=(n.value, rl.value)).copy()

    # -- GPU entry points (arrays are caller-owned; numpy or torch)
    def encode(self, frames, y_sym, y_idx=None, z_sym=None, stream=None, u8=False):
        n = ctypes.c_uint64(0)
        fn = _L.lic_encode_u8 if u8 else _L.lic_encode
        batch = frames.shape[0]
        self._chk(fn(self._h, _ptr(frames), batch, _ptr(y_sym), _ptr(y_idx), _ptr(z_sym),
                     ctypes.addressof(n) if stream is None else None, _stream(stream)), "lic_encode")
        return n.value

    def hyper_indexes(self, z_sym, y_idx, stream=None):
        self._chk(_L.lic_hyper_indexes(self._h, _ptr(z_sym), z_sym.shape[0], _ptr(y_idx), _stream(stream)),
                  "lic_hyper_indexes")

    def decode(self, y_sym, frames, stream=None, u8=False):
        fn = _L.lic_decode_u8 if u8 else _L.lic_decode
        self._chk(fn(self._h, _ptr(y_sym), y_sym.shape[0], _ptr(frames), _stream(stream)), "lic_decode")

    # -- pool
    def buf_acquire(self, nbytes):
        p = _P()
        self._chk(_L.lic_buf_acquire(self._h, nbytes, ctypes.byref(p)), "lic_buf_acquire")
        return p.value

    def buf_release(self, ptr):
        return _L.lic_buf_release(self._h, ptr)

    def buf_stats(self):
        a, r = ctypes.c_uint64(), ctypes.c_uint64()
        _L.lic_buf_stats(self._h, ctypes.byref(a), ctypes.byref(r))
        return a.value, r.value

    # -- workspace (PAPER.md:105 pooled device memory; the caller may own it)
    def workspace_bytes(self, batch=0):
        return int(_L.lic_workspace_bytes(self._h, batch))

    def bind_workspace(self, buf, nbytes=None):
        """Use caller-owned device memory (a torch tensor or a device address) as the
        codec's workspace; returns the resulting max batch.  The caller keeps `buf` alive."""
        if nbytes is None:
            nbytes = buf.numel() * buf.element_size()
        self._ws = buf                                  # keep the owner alive with the codec
        self._chk(_L.lic_bind_workspace(self._h, _ptr(buf), nbytes), "lic_bind_workspace")
        return self.max_batch_now()

    def max_batch_now(self):
        b = _u32()
        self._chk(_L.lic_max_batch(self._h, ctypes.byref(b)), "lic_max_batch")
        return b.value

    def range_count(self, reset=True):
        """Activations stored saturated to the fp16 range since the last reset (lic_range_count)."""
        n = ctypes.c_uint64()
        self._chk(_L.lic_range_count(self._h, ctypes.byref(n), int(reset)), "lic_range_count")
        return n.value

    def set_zero_copy(self, on=True):
        self._chk(_L.lic_set_zero_copy(self._h, int(on)), "lic_set_zero_copy")

    # -- measurement
    def profile(self, on=True, layers=None):
        """Bracket GEMM-engine launches with CUDA events: all layers, or only `layers` (names)."""
        if layers is None:
            self._chk(_L.lic_profile(self._h, int(on)), "lic_profile")
        else:
            mask = 0
            for n in layers:
                mask |= 1 << LAYERS.index(n)
            self._chk(_L.lic_profile_layers(self._h, mask if on else 0), "lic_profile_layers")

    def profile_read(self):
        """{layer: (ms, launches)} accumulated since profile(True); resets."""
        out = {}
        for i, name in enumerate(LAYERS):
            ms, n = ctypes.c_double(), ctypes.c_uint64()
            if _L.lic_profile_read(self._h, i, ctypes.byref(ms), ctypes.byref(n)) == 0 and n.value:
                out[name] = (ms.value, n.value)
        return out

    def trace(self, layer, on=True):
        lid = LAYERS.index(layer) if isinstance(layer, str) else layer
        self._chk(_L.lic_trace(self._h, lid, int(on)), "lic_trace")

    def trace_read(self):
        out = np.zeros(256 * 24, np.uint64)
        self._chk(_L.lic_trace_read(self._h, _ptr(out), out.size), "lic_trace_read")
        return out.reshape(256, 24)

    def launch_count(self):
        n = ctypes.c_uint64()
        self._chk(_L.lic_launch_count(self._h, ctypes.byref(n)), "lic_launch_count")
        return n.value

    # -- test exports
    def layer_shapes(self, layer):
        lid = LAYERS.index(layer) if isinstance(layer, str) else layer
        i, o = Shape(), Shape()
        self._chk(_L.lic_layer_shapes(self._h, lid, ctypes.byref(i), ctypes.byref(o)), "lic_layer_shapes")
        return i.tuple(), o.tuple()

    def test_layer(self, layer, x):
        """x: f32 [B, Cin, Hin, Win] numpy -> f32 [B, Cout, Hout, Wout]."""
        lid = LAYERS.index(layer) if isinstance(layer, str) else layer
        _, o = self.layer_shapes(lid)
        x = np.ascontiguousarray(x, np.float32)
        out = np.empty((x.shape[0],) + o, np.float32)
        self._chk(_L.lic_test_layer(self._h, lid, _ptr(x), x.shape[0], _ptr(out), None), "lic_test_layer")
        return out

    def test_sigma_to_index(self, sigma):
        s = np.ascontiguousarray(sigma, np.float32)
        idx = np.empty(s.shape, np.uint8)
        self._chk(_L.lic_test_sigma_to_index(self._h, _ptr(s), s.size, _ptr(idx)), "lic_test_sigma_to_index")
        return idx

    def set_debug(self, on=True):
        self._chk(_L.lic_set_debug(self._h, int(on)), "lic_set_debug")

    def debug_latents(self, batch):
        y = np.empty((batch,) + self.y_shape, np.float32)
        z = np.empty((batch,) + self.z_shape, np.float32) if self.hyper else None
        s = np.empty((batch,) + self.y_shape, np.float32) if self.hyper else None
        self._chk(_L.lic_debug_latents(self._h, batch, _ptr(y), _ptr(z), _ptr(s)), "lic_debug_latents")
        return y, z, s


class Pipeline:
    """lic_pipeline: GPU control thread (the caller) + native coder worker pool."""

    def __init__(self, codec: Codec, coder_threads: int, batch: int, inflight: int = 2, u8: bool = True,
                 serial: bool = False, keep_bitstreams: bool = False, substreams: int = 1, coder: int = 0,
                 pace_fps: float = 0.0, timeline: bool = False, coder_parts: int = 1):
        self.codec = codec
        self.substreams = substreams
        self.cfg = PipelineConfig(coder_threads, batch, inflight, int(u8), int(serial), int(keep_bitstreams),
                                  substreams, coder, float(pace_fps), int(timeline), coder_parts)
        self._h = _P()
        st = _L.lic_pipeline_open(codec.handle, ctypes.byref(self.cfg), ctypes.byref(self._h))
        if st:
            raise LicError(st, "lic_pipeline_open")

    def run(self, frames_in, frames_out, nframes=None):
        n = nframes if nframes is not None else frames_in.shape[0]
        st = PipelineStats()
        rc = _L.lic_pipeline_run(self._h, _ptr(frames_in), n, _ptr(frames_out), ctypes.byref(st))
        if rc:
            raise LicError(rc, "lic_pipeline_run: " + (_L.lic_last_error(self.codec.handle) or b"").decode())
        return st.as_dict()

    def timeline(self):
        """lic_pipeline_timeline: list of dicts (kind name, lane, batch, frame, ready / start / end ms)."""
        n = _sz()
        self._chk_rc(_L.lic_pipeline_timeline(self._h, None, 0, ctypes.byref(n)), "lic_pipeline_timeline")
        buf = (TimelineEvent * max(1, n.value))()
        self._chk_rc(_L.lic_pipeline_timeline(self._h, buf, n.value, ctypes.byref(n)), "lic_pipeline_timeline")
        return [dict(kind=TIMELINE_KINDS[e.kind], lane=e.lane, batch=e.batch, frame=e.frame, ready=e.t_ready_ms,
                     start=e.t_start_ms, end=e.t_end_ms) for e in buf[:n.value]]

    @staticmethod
    def _chk_rc(rc, what):
        if rc:
            raise LicError(rc, what)

    def bitstream(self, i):
        y, z = ctypes.POINTER(ctypes.c_uint8)(), ctypes.POINTER(ctypes.c_uint8)()
        yl, zl = ctypes.c_size_t(), ctypes.c_size_t()
        rc = _L.lic_pipeline_bitstream(self._h, i, ctypes.byref(y), ctypes.byref(yl), ctypes.byref(z),
                                       ctypes.byref(zl))
        if rc:
            raise LicError(rc, "lic_pipeline_bitstream")
        yb = ctypes.string_at(y, yl.value)
        zb = ctypes.string_at(z, zl.value) if zl.value else None
        return yb, zb

    def close(self):
        if self._h:
            _L.lic_pipeline_close(self._h)
            self._h = _P()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
