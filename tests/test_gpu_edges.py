"""Edge cases of the CUDA path against the oracle (-m gpu): partial batches, the smallest
geometries (one y / z element per channel), and saturating latents (the +-L clamp and its
counter)."""
import numpy as np
import pytest

from lic_synth import ModelSpec, generate_weights, synth_frames_u8, u8_to_f32_chw, write_licw
from oracle import oracle as O

from parity import check_float, check_indexes, check_symbols

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def lic():
    from paper_2208_01641_b200 import lic as L
    return L


def _encode(c, frames, hyper, u8=True):
    B = frames.shape[0]
    ys = np.empty((B,) + c.y_shape, np.int8)
    yi = np.empty((B,) + c.y_shape, np.uint8) if hyper else None
    zs = np.empty((B,) + c.z_shape, np.int8) if hyper else None
    nsat = c.encode(np.ascontiguousarray(frames), ys, yi, zs, u8=u8)
    return ys, yi, zs, nsat


@pytest.mark.parametrize("kind", [1, 0])
def test_partial_batches_are_per_frame_identical(lic, kind):
    """A frame's symbols, indexes and reconstruction do not depend on the batch it is coded
    in (batch 3 of max 3, batch 1, batch 2)."""
    spec = ModelSpec(kind=kind, N=128, M=192)
    c = lic.Codec(write_licw(spec, generate_weights(spec, seed=0)), 136, 200, max_batch=3)
    fr = synth_frames_u8(3, 136, 200, seed=31)
    hyper = kind == 1
    y3, i3, z3, _ = _encode(c, fr, hyper)
    y1, i1, z1, _ = _encode(c, fr[2:3], hyper)
    y2, i2, z2, _ = _encode(c, fr[:2], hyper)
    assert np.array_equal(y1[0], y3[2]) and np.array_equal(y2, y3[:2])
    if hyper:
        assert np.array_equal(i1[0], i3[2]) and np.array_equal(i2, i3[:2])
        assert np.array_equal(z1[0], z3[2]) and np.array_equal(z2, z3[:2])
        ix = np.empty_like(i3[:1])
        c.hyper_indexes(z3[1:2], ix)
        assert np.array_equal(ix[0], i3[1])
    d3 = np.empty((3, 136, 200, 3), np.uint8)
    d1 = np.empty((1, 136, 200, 3), np.uint8)
    c.decode(y3, d3, u8=True)
    c.decode(y3[1:2], d1, u8=True)
    assert np.array_equal(d1[0], d3[1])
    c.close()


@pytest.mark.parametrize("kind,H,W", [(1, 8, 8), (0, 8, 8), (1, 2, 2), (0, 16, 16), (1, 16, 48)])
def test_smallest_geometries(lic, kind, H, W):
    """Frames that pad to a single 64 x 64 (hyper: y 4 x 4, z 1 x 1) or 16 x 16 (factorized:
    y 1 x 1) block (W = 16, 48: rows of 3W bytes a multiple of 16 -- the row-halo g_a L1): encode, indexes and decode against the oracle."""
    spec = ModelSpec(kind=kind, N=128, M=192)
    w = generate_weights(spec, seed=0)
    hyper = kind == 1
    c = lic.Codec(write_licw(spec, w), H, W, max_batch=1)
    fr = synth_frames_u8(1, H, W, seed=5)
    x = u8_to_f32_chw(fr)
    c.set_debug(True)
    ys, yi, zs, _ = _encode(c, fr, hyper)
    y, z, _ = c.debug_latents(1)
    xp, crop = O.pad_chw(x[0], hyper=hyper)
    p = O.encode_planes(xp, w, hyper, 32)
    check_float(y[0], p["y"], what="tiny y")
    mu = 0.0 if hyper else w["mu_y"][:, None, None]
    check_symbols(ys[0], p["y_sym"], p["y"] - mu, what="tiny y_sym")
    if hyper:
        check_float(z[0], p["z"], what="tiny z")
        nz = check_symbols(zs[0], p["z_sym"], p["z"] - w["mu_z"][:, None, None], what="tiny z_sym")
        assert nz == 0, "z symbol at a tie: indexes not comparable"
        check_indexes(yi[0], p["y_idx"], p["sigma"], w["scale_table"], what="tiny y_idx")
    out = np.empty((1, 3, H, W), np.float32)
    c.decode(p["y_sym"][None], out)
    check_float(out[0], O.decode_frame(p["y_sym"], w, hyper, crop, H, W), what="tiny x-hat")
    c.close()


def test_saturating_latents_clamp_and_count(lic):
    """A g_a L4 scaled by 64 (a power of two: the weights stay fp16-exact) drives |y - mu|
    past L = 32 on ~15 % of the elements: the symbols are the clamped oracle values and the
    saturation counter matches the oracle's count."""
    spec = ModelSpec(kind=0, N=128, M=192)
    w = generate_weights(spec, seed=0)
    w["ga4.w"] = (w["ga4.w"] * 64).astype(np.float32)
    H, W = 64, 96
    c = lic.Codec(write_licw(spec, w), H, W, max_batch=1)
    fr = synth_frames_u8(1, H, W, seed=9)
    c.set_debug(True)
    ys, _, _, nsat = _encode(c, fr, False)
    y, _, _ = c.debug_latents(1)
    xp, _ = O.pad_chw(u8_to_f32_chw(fr)[0], hyper=False)
    p = O.encode_planes(xp, w, False, 32)
    assert p["n_sat"] > 100                                   # the case is really saturating
    rel = np.abs(y[0] - p["y"]) / np.maximum(1.0, np.abs(p["y"]))
    assert float(rel.max()) <= 1e-3                           # latents up to ~90: relative bar
    check_symbols(ys[0], p["y_sym"], p["y"] - w["mu_y"][:, None, None], what="saturated y_sym")
    assert abs(int(nsat) - int(p["n_sat"])) <= 1
    assert int(np.abs(ys[0].astype(np.int32)).max()) == 32
    c.close()
