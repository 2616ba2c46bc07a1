"""Kernel-variant equivalence on the GPU (-m gpu): the experiment switches of DESIGN.md §7 that
change how a layer is computed but not what it computes.

- g_a L1 on u8 frames as a row halo with five K = 16 MMAs (default, R16g) or as im2col
  tiles whose raw u8 patch comes by one TMA box per tile (3W % 16 == 0) or by 4-byte cp.async:
  the same products in the same K-step order, so the latents are bit-identical; likewise 4
  hi-only A stages vs 2 split ones, and split-K h layers vs single-pass ones (up to summation
  order: compared with the oracle bars).
- the two-group GDN / IGDN epilogue (y from the norm operand and the signs, R16e) vs
  the single-group one (x kept in registers): different rounding, both within the oracle bars.
"""
import contextlib
import os

import numpy as np
import pytest

from lic_synth import ModelSpec, generate_weights, synth_frames_u8, u8_to_f32_chw, write_licw
from oracle import oracle as O

from parity import check_float, check_symbols

pytestmark = pytest.mark.gpu

SPEC = ModelSpec(kind=1, N=128, M=192)
H, W = 130, 320          # 3W = 960: TMA-eligible rows; 130 rows: ragged bottom tiles


@pytest.fixture(scope="module")
def lic():
    from paper_2208_01641_b200 import lic as L
    return L


@pytest.fixture(scope="module")
def data():
    w = generate_weights(SPEC, seed=0)
    fr = synth_frames_u8(2, H, W, seed=21)
    x = u8_to_f32_chw(fr)
    planes = []
    for b in range(2):
        xp, crop = O.pad_chw(x[b], hyper=True)
        planes.append((O.encode_planes(xp, w, True, 32), crop))
    return dict(w=w, blob=write_licw(SPEC, w), fr=fr, planes=planes)


@contextlib.contextmanager
def env(**kv):
    old = {k: os.environ.get(k) for k in kv}
    os.environ.update({k: str(v) for k, v in kv.items()})
    try:
        yield
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


def run(lic, data, **kv):
    with env(**kv):
        c = lic.Codec(data["blob"], H, W, max_batch=2)
    try:
        ys = np.empty((2,) + c.y_shape, np.int8)
        yi = np.empty((2,) + c.y_shape, np.uint8)
        zs = np.empty((2,) + c.z_shape, np.int8)
        c.set_debug(True)
        c.encode(np.ascontiguousarray(data["fr"]), ys, yi, zs, u8=True)
        y, z, _ = c.debug_latents(2)
        xh = np.empty((2, 3, H, W), np.float32)
        c.decode(np.stack([p["y_sym"] for p, _ in data["planes"]]), xh)
        return dict(y=y.copy(), z=z.copy(), ys=ys, yi=yi, zs=zs, xh=xh)
    finally:
        c.close()


def test_raw_patch_tma_vs_cp_async(lic, data):
    a = run(lic, data)                                  # row halo (R16g)
    b = run(lic, data, LIC_RAW_TMA=0)                   # im2col, 4-byte cp.async
    c = run(lic, data, LIC_RAW_TMA=0, LIC_L1_STAGES=0)  # im2col, cp.async, 2 split stages
    d = run(lic, data, LIC_L1_ROWS=0)                   # im2col, TMA boxes, 4 hi-only stages
    for k in ("y", "z", "ys", "yi", "zs", "xh"):
        assert np.array_equal(a[k], b[k]), k
        assert np.array_equal(a[k], c[k]), k
        assert np.array_equal(a[k], d[k]), k


@pytest.mark.parametrize("g2", [0, 1, 2])
def test_gdn_epilogue_variants_vs_oracle(lic, data, g2):
    r = run(lic, data, LIC_G2=g2)
    w = data["w"]
    for f in range(2):
        p, crop = data["planes"][f]
        ey = check_float(r["y"][f], p["y"], what=f"G2={g2} y")
        check_symbols(r["ys"][f], p["y_sym"], p["y"], what=f"G2={g2} y_sym")
        ref = O.decode_frame(p["y_sym"], w, True, crop, H, W)
        ex = check_float(r["xh"][f], ref, what=f"G2={g2} x-hat")
        print(f"G2={g2} frame {f}: y max-abs {ey:.2e}, x-hat max-abs {ex:.2e}")


@pytest.mark.parametrize("g2_192", [0, 1])
def test_n192_two_group_chunked_norm_vs_oracle(lic, g2_192):
    """N = 192 codec (C4 / C5 shapes): the two-group epilogue with the norm in three 64-column
    chunks (LIC_G2_192=1) and the single-group one both meet the oracle bars."""
    spec = ModelSpec(kind=1, N=192, M=320)
    Hh, Ww = 128, 192
    w = generate_weights(spec, seed=0)
    fr = synth_frames_u8(1, Hh, Ww, seed=23)
    x = u8_to_f32_chw(fr)
    xp, crop = O.pad_chw(x[0], hyper=True)
    pl = O.encode_planes(xp, w, True, 32)
    with env(LIC_G2_192=g2_192):
        c = lic.Codec(write_licw(spec, w), Hh, Ww, max_batch=1)
    try:
        ys = np.empty((1,) + c.y_shape, np.int8)
        yi = np.empty((1,) + c.y_shape, np.uint8)
        zs = np.empty((1,) + c.z_shape, np.int8)
        c.set_debug(True)
        c.encode(np.ascontiguousarray(fr), ys, yi, zs, u8=True)
        y, _, _ = c.debug_latents(1)
        ey = check_float(y[0], pl["y"], what=f"N=192 G2_192={g2_192} y")
        check_symbols(ys[0], pl["y_sym"], pl["y"], what="N=192 y_sym")
        xh = np.empty((1, 3, Hh, Ww), np.float32)
        c.decode(pl["y_sym"][None], xh)
        ref = O.decode_frame(pl["y_sym"], w, True, crop, Hh, Ww)
        ex = check_float(xh[0], ref, what=f"N=192 G2_192={g2_192} x-hat")
        print(f"N=192 G2_192={g2_192}: y max-abs {ey:.2e}, x-hat max-abs {ex:.2e}")
    finally:
        c.close()
