"""Python face of the CPU oracle (``oracle/lic_oracle.c``).

TEST INFRASTRUCTURE ONLY: may be imported only by ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` / ``--impl
reference`` legs.  It never imports the product package and the product never
imports it.  It composes the C primitives in the paper's order (Fig. 1,
§III.A-B) with no fusion or reordering; numpy is used
only for data movement (padding, cropping, reshapes) and to hold arrays.

Parity status: every primitive is pinned by tests/test_oracle_*.py; the whole
network composition is pinned against an independent torch-float64 composition
(tests/test_oracle_network.py) plus latent fidelity and determinism.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_SRC = os.path.join(_HERE, "lic_oracle.c")

OR_OK, OR_EINVAL, OR_ECORRUPT, OR_ENOSPACE = 0, 1, 3, 5


def build_oracle(force: bool = False) -> str:
    """Compile the oracle (gcc, -O2, no fast-math so fp64 semantics hold)."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-std=c11",
                               "-o", _SO, _SRC, "-lm"])
    return _SO


_lib = None


def lib():
    global _lib
    if _lib is None:
        build_oracle()
        L = ctypes.CDLL(_SO)
        P = ctypes.c_void_p
        i, sz = ctypes.c_int, ctypes.c_size_t
        L.or_conv2d.argtypes = [P, i, i, i, P, P, i, i, i, i, P]
        L.or_deconv2d.argtypes = [P, i, i, i, P, P, i, i, i, i, i, P]
        L.or_gdn.argtypes = [P, i, i, i, P, P, i, P]
        L.or_onedn.argtypes = [P, i, i, i, P, P, i, P]
        L.or_quantize.argtypes = [P, i, i, i, P, i, P, P, P]
        L.or_dequantize.argtypes = [P, i, i, i, P, P]
        L.or_scale_index.argtypes = [P, sz, P, i, P]
        L.or_cdf_row.argtypes = [ctypes.c_double, i, P]
        L.or_rans_encode.argtypes = [P, P, sz, P, i, i, i, P, sz, ctypes.POINTER(sz)]
        L.or_rans_decode.argtypes = [P, sz, P, sz, P, i, i, i, P]
        _lib = L
    return _lib


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p) if a is not None else None


def _f32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


# ---------------------------------------------------------------- primitives
def conv2d(x, w, b, stride, pad):
    """SPEC.md:43-46 (see lic_oracle.c or_conv2d)."""
    x, w, b = _f32(x), _f32(w), _f32(b)
    cin, H, W = x.shape
    cout, cin2, k, _ = w.shape
    assert cin == cin2
    Ho, Wo = (H + 2 * pad - k) // stride + 1, (W + 2 * pad - k) // stride + 1
    out = np.empty((cout, Ho, Wo), np.float32)
    rc = lib().or_conv2d(_p(x), cin, H, W, _p(w), _p(b), cout, k, stride, pad, _p(out))
    if rc:
        raise ValueError("or_conv2d")
    return out


def deconv2d(x, w, b, stride, pad, output_padding):
    """SPEC.md:53-56 + SURVEY.md c2 (see lic_oracle.c or_deconv2d); w is out x in x k x k."""
    x, w, b = _f32(x), _f32(w), _f32(b)
    cin, H, W = x.shape
    cout, cin2, k, _ = w.shape
    assert cin == cin2
    Ho = (H - 1) * stride - 2 * pad + k + output_padding
    Wo = (W - 1) * stride - 2 * pad + k + output_padding
    out = np.empty((cout, Ho, Wo), np.float32)
    rc = lib().or_deconv2d(_p(x), cin, H, W, _p(w), _p(b), cout, k, stride, pad,
                           output_padding, _p(out))
    if rc:
        raise ValueError("or_deconv2d")
    return out


def gdn(x, beta, gamma, inverse=False):
    """SPEC.md:66 (see lic_oracle.c or_gdn)."""
    x = _f32(x)
    C, H, W = x.shape
    out = np.empty_like(x)
    rc = lib().or_gdn(_p(x), C, H, W, _p(_f32(beta)), _p(_f32(gamma)), int(inverse), _p(out))
    if rc:
        raise ValueError("or_gdn")
    return out


def onedn(x, beta, gamma, inverse=False):
    """SPEC.md:76 (see lic_oracle.c or_onedn)."""
    x = _f32(x)
    C, H, W = x.shape
    out = np.empty_like(x)
    rc = lib().or_onedn(_p(x), C, H, W, _p(_f32(beta)), _p(_f32(gamma)), int(inverse), _p(out))
    if rc:
        raise ValueError("or_onedn")
    return out


def relu(x):
    """max(x, 0) (SPEC.md:319 h_a/h_s activations)."""
    return np.maximum(_f32(x), np.float32(0.0))


def quantize(y, mu, L):
    """SPEC.md:191-199 (see lic_oracle.c or_quantize). Returns (sym int8, yhat f32, n_sat)."""
    y = _f32(y)
    C, H, W = y.shape
    sym = np.empty(y.shape, np.int8)
    yhat = np.empty_like(y)
    nsat = ctypes.c_uint64(0)
    rc = lib().or_quantize(_p(y), C, H, W, _p(_f32(mu)) if mu is not None else None, L,
                           _p(sym), _p(yhat), ctypes.byref(nsat))
    if rc:
        raise ValueError("or_quantize")
    return sym, yhat, int(nsat.value)


def dequantize(sym, mu):
    sym = np.ascontiguousarray(sym, dtype=np.int8)
    C, H, W = sym.shape
    out = np.empty(sym.shape, np.float32)
    lib().or_dequantize(_p(sym), C, H, W, _p(_f32(mu)) if mu is not None else None, _p(out))
    return out


def scale_index(sigma, table):
    """SPEC.md:181-189, SURVEY.md c10 (see lic_oracle.c or_scale_index)."""
    s = _f32(sigma)
    t = _f32(table)
    idx = np.empty(s.shape, np.uint8)
    rc = lib().or_scale_index(_p(s), s.size, _p(t), t.size, _p(idx))
    if rc:
        raise ValueError("or_scale_index")
    return idx


def cdf_row(sigma, L):
    """SURVEY.md §8(c) step 9 (see lic_oracle.c or_cdf_row)."""
    out = np.empty(2 * L + 2, np.uint32)
    rc = lib().or_cdf_row(float(sigma), int(L), _p(out))
    if rc:
        raise ValueError("or_cdf_row")
    return out


def cdf_table(sigmas, L):
    return np.stack([cdf_row(float(s), L) for s in np.asarray(sigmas, np.float32)])


def rans_encode(sym, rows, cdf, sym_min=None):
    """SURVEY.md §8(c) step 10 (see lic_oracle.c or_rans_encode).  sym/rows flat;
    sym_min defaults to -L for codec tables (row_len = 2L+2)."""
    sym = np.ascontiguousarray(sym, dtype=np.int8).ravel()
    rows = np.ascontiguousarray(rows, dtype=np.int32).ravel()
    cdf = np.ascontiguousarray(cdf, dtype=np.uint32)
    cap = 2 * sym.size + 16
    out = np.empty(cap, np.uint8)
    n = ctypes.c_size_t(0)
    if sym_min is None:
        sym_min = -((cdf.shape[1] - 2) // 2)
    rc = lib().or_rans_encode(_p(sym), _p(rows), sym.size, _p(cdf), cdf.shape[0], cdf.shape[1],
                              int(sym_min), _p(out), cap, ctypes.byref(n))
    if rc:
        raise ValueError(f"or_rans_encode rc={rc}")
    return out[: n.value].tobytes()


class CorruptStream(Exception):
    pass


def rans_decode(data, rows, cdf, sym_min=None):
    rows = np.ascontiguousarray(rows, dtype=np.int32).ravel()
    cdf = np.ascontiguousarray(cdf, dtype=np.uint32)
    buf = np.frombuffer(bytes(data), np.uint8) if len(data) else np.zeros(1, np.uint8)
    sym = np.empty(rows.size, np.int8)
    if sym_min is None:
        sym_min = -((cdf.shape[1] - 2) // 2)
    rc = lib().or_rans_decode(_p(buf), len(data), _p(rows), rows.size, _p(cdf), cdf.shape[0],
                              cdf.shape[1], int(sym_min), _p(sym))
    if rc == OR_ECORRUPT:
        raise CorruptStream()
    if rc:
        raise ValueError(f"or_rans_decode rc={rc}")
    return sym


def slab_bounds(C, K):
    """Channel slab k = [floor(k*C/K), floor((k+1)*C/K)) (R21)."""
    return [(k * C // K, (k + 1) * C // K) for k in range(K)]


def rans_encode_slabs(sym_chw, rows_chw, cdf, K):
    """K channel-slab substreams (R21): each slab an independent step-10 string;
    K = 1 is the plain string, K > 1 is K big-endian u32 lengths followed by the strings.
    rows_chw None: the row of a symbol is its channel."""
    sym_chw = np.asarray(sym_chw)
    C = sym_chw.shape[0]
    if K == 1:
        rows = channel_rows(sym_chw.shape) if rows_chw is None else np.asarray(rows_chw, np.int32).ravel()
        return rans_encode(sym_chw, rows, cdf)
    parts = []
    for c0, c1 in slab_bounds(C, K):
        sub = sym_chw[c0:c1]
        if rows_chw is None:
            rows = channel_rows(sub.shape) + c0
        else:
            rows = np.asarray(rows_chw[c0:c1], np.int32).ravel()
        parts.append(rans_encode(sub, rows, cdf))
    head = b"".join(len(p).to_bytes(4, "big") for p in parts)
    return head + b"".join(parts)


def rans_decode_slabs(data, shape, rows_chw, cdf, K):
    """Inverse of rans_encode_slabs; CorruptStream on a bad framing."""
    C, H, W = shape
    if K == 1:
        rows = channel_rows(shape) if rows_chw is None else np.asarray(rows_chw, np.int32).ravel()
        return rans_decode(data, rows, cdf).reshape(shape)
    data = bytes(data)
    if len(data) < 4 * K:
        raise CorruptStream()
    lens = [int.from_bytes(data[4 * k:4 * k + 4], "big") for k in range(K)]
    if 4 * K + sum(lens) != len(data):
        raise CorruptStream()
    out = np.empty(shape, np.int8)
    pos = 4 * K
    for (c0, c1), n in zip(slab_bounds(C, K), lens):
        sub_shape = (c1 - c0, H, W)
        if rows_chw is None:
            rows = channel_rows(sub_shape) + c0
        else:
            rows = np.asarray(rows_chw[c0:c1], np.int32).ravel()
        out[c0:c1] = rans_decode(data[pos:pos + n], rows, cdf).reshape(sub_shape)
        pos += n
    return out


def channel_rows(shape):
    """Row index per symbol of a C x H x W plane coded with per-channel tables."""
    C, H, W = shape
    return np.repeat(np.arange(C, dtype=np.int32), H * W)


# ---------------------------------------------------------------- geometry
def padded_size(H, W, hyper):
    """centred zero pad to a multiple of 16 (fact) / 64 (hyper)."""
    P = 64 if hyper else 16
    return -(-H // P) * P, -(-W // P) * P


def pad_offsets(H, W, hyper):
    Hp, Wp = padded_size(H, W, hyper)
    return Hp, Wp, (Hp - H) // 2, (Wp - W) // 2


def ingest_u8(frame_hwc_u8, hyper):
    """x = float(u8)/255 (fp32 IEEE division), CHW, centred
    zero pad.  Returns (x padded CHW f32, (top, left))."""
    H, W, _ = frame_hwc_u8.shape
    x = np.moveaxis(frame_hwc_u8, -1, 0).astype(np.float32) / np.float32(255.0)
    return pad_chw(x, hyper)


def pad_chw(x, hyper):
    C, H, W = x.shape
    Hp, Wp, top, left = pad_offsets(H, W, hyper)
    out = np.zeros((C, Hp, Wp), np.float32)
    out[:, top:top + H, left:left + W] = x
    return out, (top, left)


# ---------------------------------------------------------------- transforms
def _norm(act):
    """Activation of g_a / g_s: 0 GDN, 1 1DN (the paper's
    implementation C)."""
    return onedn if act == 1 else gdn


def g_a(x, w, act=0):
    """g_a: conv5s2 -> GDN (or 1DN) x3 -> conv5s2 N->M."""
    h = x
    for i in (1, 2, 3):
        h = conv2d(h, w[f"ga{i}.w"], w[f"ga{i}.b"], 2, 2)
        h = _norm(act)(h, w[f"ga{i}.beta"], w[f"ga{i}.gamma"], inverse=False)
    return conv2d(h, w["ga4.w"], w["ga4.b"], 2, 2)


def g_s(yhat, w, act=0):
    """g_s: deconv5s2 (output_padding 1) -> IGDN (or inverse 1DN) x3 -> deconv N->3."""
    h = yhat
    for i in (1, 2, 3):
        h = deconv2d(h, w[f"gs{i}.w"], w[f"gs{i}.b"], 2, 2, 1)
        h = _norm(act)(h, w[f"gs{i}.beta"], w[f"gs{i}.gamma"], inverse=True)
    return deconv2d(h, w["gs4.w"], w["gs4.b"], 2, 2, 1)


def h_a(y, w):
    """h_a (SPEC.md:319, :336 input |y|): conv3s1, ReLU, conv5s2, ReLU, conv5s2."""
    h = conv2d(np.abs(_f32(y)), w["ha1.w"], w["ha1.b"], 1, 1)
    h = relu(h)
    h = conv2d(h, w["ha2.w"], w["ha2.b"], 2, 2)
    h = relu(h)
    return conv2d(h, w["ha3.w"], w["ha3.b"], 2, 2)


def h_s(zhat, w):
    """h_s: deconv5s2, ReLU, deconv5s2, ReLU, conv3s1 N->M, ReLU."""
    h = relu(deconv2d(zhat, w["hs1.w"], w["hs1.b"], 2, 2, 1))
    h = relu(deconv2d(h, w["hs2.w"], w["hs2.b"], 2, 2, 1))
    return relu(conv2d(h, w["hs3.w"], w["hs3.b"], 1, 1))


# ---------------------------------------------------------------- codecs
@dataclass
class Tables:
    fact_y: np.ndarray | None     # M x (2L+2): per-channel y rows (factorized)
    z: np.ndarray | None          # N x (2L+2): per-channel z rows (hyper)
    gauss: np.ndarray | None      # 64 x (2L+2): scale-table rows (hyper)


def build_tables(w, hyper, L):
    if hyper:
        return Tables(None, cdf_table(w["sigma_z"], L), cdf_table(w["scale_table"], L))
    return Tables(cdf_table(w["sigma_y"], L), None, None)


def encode_planes(x_pad, w, hyper, L, act=0):
    """GPU half of encode: returns the latents and planes."""
    y = g_a(x_pad, w, act)
    out = {"y": y}
    if not hyper:
        sym, yhat, nsat = quantize(y, w["mu_y"], L)
        out.update(y_sym=sym, yhat=yhat, n_sat=nsat)
        return out
    z = h_a(y, w)
    zs, zhat, nsat_z = quantize(z, w["mu_z"], L)
    sigma = h_s(zhat, w)
    idx = scale_index(sigma, w["scale_table"])
    ys, yhat, nsat_y = quantize(y, None, L)
    out.update(z=z, z_sym=zs, zhat=zhat, sigma=sigma, y_idx=idx, y_sym=ys, yhat=yhat,
               n_sat=nsat_y + nsat_z)
    return out


def code_planes(planes, tables, hyper, substreams=1):
    """CPU half of encode: rANS strings; the y string as `substreams`
    channel slabs (R21; 1 = one plain string)."""
    ys = planes["y_sym"]
    if not hyper:
        return rans_encode_slabs(ys, None, tables.fact_y, substreams), None
    yb = rans_encode_slabs(ys, planes["y_idx"], tables.gauss, substreams)
    zs = planes["z_sym"]
    zb = rans_encode(zs, channel_rows(zs.shape), tables.z)
    return yb, zb


def hyper_indexes(z_sym, w):
    """Decoder GPU1: z symbols -> z-hat -> h_s -> y CDF indexes."""
    zhat = dequantize(z_sym, w["mu_z"])
    return scale_index(h_s(zhat, w), w["scale_table"])


def decode_frame(y_sym, w, hyper, crop, H, W, act=0):
    """Decoder GPU2: y-hat = s + mu (hyper mu = 0), x-hat =
    clamp(g_s(y-hat), 0, 1), cropped by the pad offsets."""
    yhat = dequantize(y_sym, None if hyper else w["mu_y"])
    xh = np.clip(g_s(yhat, w, act), np.float32(0.0), np.float32(1.0))
    top, left = crop
    return np.ascontiguousarray(xh[:, top:top + H, left:left + W])


def decode_strings(yb, zb, w, tables, hyper, y_shape, z_shape, crop, H, W, substreams=1, act=0):
    """Full decode: CPU1 rANS(z) -> GPU1 h_s -> CPU2 rANS(y) -> GPU2 g_s."""
    if hyper:
        zs = rans_decode(zb, channel_rows(z_shape), tables.z).reshape(z_shape)
        idx = hyper_indexes(zs, w)
        ys = rans_decode_slabs(yb, y_shape, idx, tables.gauss, substreams)
    else:
        ys = rans_decode_slabs(yb, y_shape, None, tables.fact_y, substreams)
    return decode_frame(ys, w, hyper, crop, H, W, act), ys
