"""Precision edges of the graded split-FP16 mode and the caller-owned workspace (-m gpu).

* Weights: the tensor cores take fp16 operands, so lic_open rejects conv / deconv weights
  and gamma that are not exactly representable in fp16 (LIC_EINVAL with a message) instead
  of rounding them silently (R16).
* Large activations (R16d): the GDN / IGDN norm operand x^2 is split into fp16
  hi + lo, whose range ends at 65504 (|x| = 256).  Each pixel scales it by an exact power of
  two, so layers whose activations pass 256 still match the oracle (SPEC.md:66 GDN).
  Activations themselves beyond +-65504 (the range of the paper's FP16 engines,
  PAPER.md:129) are stored saturated and counted by lic_range_count -- never inf / NaN.
* Workspace (PAPER.md:105 pooled device memory): a torch-owned block bound with
  lic_bind_workspace gives bit-identical planes and frames.
"""
import numpy as np
import pytest

from lic_synth import ModelSpec, generate_weights, synth_frames_u8, write_licw
from oracle import oracle as O

from parity import check_float, check_indexes, check_symbols

pytestmark = pytest.mark.gpu

HYPER = ModelSpec(kind=1, N=128, M=192)


@pytest.fixture(scope="module")
def lic():
    from paper_2208_01641_b200 import lic as L
    return L


@pytest.fixture(scope="module")
def w():
    return generate_weights(HYPER, seed=0)


# ---------------------------------------------------------------- weights
@pytest.mark.parametrize("block", ["ga2.w", "gs3.w", "ha1.w", "hs3.w", "gs1.gamma"])
def test_non_fp16_weights_rejected(lic, w, block):
    bad = {k: v.copy() for k, v in w.items()}
    flat = bad[block].reshape(-1)
    v = float(flat[7])
    flat[7] = np.float32(v * (1 + 2.0 ** -13)) if v else np.float32(1e-6)      # off the fp16 grid
    assert np.float32(np.float16(flat[7])) != flat[7]
    with pytest.raises(lic.LicError) as e:
        lic.Codec(write_licw(HYPER, bad), 64, 64)
    assert e.value.status == lic.LIC_EINVAL
    assert block in str(e.value) and "fp16" in str(e.value)


def test_fp16_overflowing_weight_rejected(lic, w):
    bad = {k: v.copy() for k, v in w.items()}
    bad["gs4.w"].reshape(-1)[0] = np.float32(1e5)            # beyond fp16's 65504
    with pytest.raises(lic.LicError) as e:
        lic.Codec(write_licw(HYPER, bad), 64, 64)
    assert e.value.status == lic.LIC_EINVAL


# ---------------------------------------------------------------- large activations
def test_gdn_layer_large_activations(lic, w):
    """g_a L2 on inputs ~200x the codec's scale: conv outputs up to ~1e3, x^2 up to ~1e6
    (beyond fp16) -- per-pixel scaled norm operand; GDN output is bounded, abs bar 1e-3."""
    c = lic.Codec(write_licw(HYPER, w), 128, 128)
    (ci, hi, wi), _ = c.layer_shapes("ga2")
    rng = np.random.default_rng(3)
    x = (rng.standard_normal((1, ci, hi, wi)) * 200).astype(np.float32)
    got = c.test_layer("ga2", x)
    pre = O.conv2d(x[0], w["ga2.w"], w["ga2.b"], 2, 2)
    assert float(np.abs(pre).max()) > 256                       # the case needs the scaling
    ref = O.gdn(pre, w["ga2.beta"], w["ga2.gamma"])
    e = check_float(got[0], ref, what="ga2 large")
    assert c.range_count() == 0
    print(f"ga2 |x| max {np.abs(pre).max():.0f}: max-abs {e:.2e}")
    c.close()


def test_igdn_layer_large_activations(lic, w):
    """g_s L3 with pre-IGDN |x| up to ~300 (x^2 ~ 1e5 > 65504) and outputs below 65504.
    IGDN multiplies the conv output's absolute error by sqrt(n) (~100 here) while the oracle
    accumulates in fp64, so the bar is normwise: max |got - ref| <= 1e-5 max |ref| (before the
    per-pixel scaling the overflowing x^2 made the output inf / NaN)."""
    c = lic.Codec(write_licw(HYPER, w), 128, 128)
    (ci, hi, wi), _ = c.layer_shapes("gs3")
    rng = np.random.default_rng(4)
    x = (rng.standard_normal((1, ci, hi, wi)) * 60).astype(np.float32)
    got = c.test_layer("gs3", x)
    pre = O.deconv2d(x[0], w["gs3.w"], w["gs3.b"], 2, 2, 1)
    ref = O.gdn(pre, w["gs3.beta"], w["gs3.gamma"], inverse=True)
    assert float(np.abs(pre).max()) > 256 and float(np.abs(ref).max()) < 65504
    e = float(np.abs(got[0].astype(np.float64) - ref).max() / np.abs(ref).max())
    assert np.all(np.isfinite(got)) and e <= 1e-5, e
    assert c.range_count() == 0
    print(f"gs3 |x| max {np.abs(pre).max():.0f}, |y| max {np.abs(ref).max():.0f}: normwise {e:.2e}")
    c.close()


def _sym_plane(c, rng, k):
    return rng.choice(np.array([-k, k], np.int8), size=(1,) + c.y_shape).astype(np.int8)


def test_decode_large_symbols_matches_oracle(lic, w):
    """A legal y plane of +-4 symbols (seed 12) drives g_s L3's pre-IGDN activations to ~410
    (x^2 past fp16) while every activation stays inside +-65504 (max ~54k): nothing saturates,
    every g_s layer on the oracle's input is within 1e-5 normwise (before the per-pixel
    scaling g_s L3 returned inf / NaN), and x-hat stays within 1e-2 of the oracle.  (x-hat's
    bar is looser than the codec's 1e-3: g_s L4 sums activations of ~5e4 into values in
    [0, 1], so the fp32-accumulation error of the activations, ~7e-6 normwise against the
    oracle's fp64 accumulation, is amplified ~1e3 -- conditioning, not the format.)"""
    H, W = 128, 192
    c = lic.Codec(write_licw(HYPER, w), H, W)
    ys = _sym_plane(c, np.random.default_rng(12), 4)
    g = ys[0].astype(np.float32)
    for i in (1, 2, 3):
        ref = O.gdn(O.deconv2d(g, w[f"gs{i}.w"], w[f"gs{i}.b"], 2, 2, 1), w[f"gs{i}.beta"], w[f"gs{i}.gamma"],
                    inverse=True)
        got = c.test_layer(f"gs{i}", g[None])[0]
        e = float(np.abs(got.astype(np.float64) - ref).max() / np.abs(ref).max())
        print(f"gs{i} on the oracle's input: |y| max {np.abs(ref).max():.0f}, normwise {e:.2e}")
        assert np.all(np.isfinite(got)) and e <= 1e-5
        g = ref
    out = np.empty((1, 3, H, W), np.float32)
    c.range_count(reset=True)
    c.decode(ys, out)
    assert c.range_count() == 0
    ref = O.decode_frame(ys[0], w, True, O.pad_offsets(H, W, True)[2:], H, W)
    err = np.abs(out[0] - ref)
    print(f"+-4 plane: x-hat max-abs {err.max():.2e}, {np.mean(err <= 1e-3):.4f} of samples within 1e-3")
    assert np.all(np.isfinite(out)) and float(err.max()) <= 1e-2
    c.close()


def test_decode_saturated_symbols_counted_and_finite(lic, w):
    """The fully saturated plane (every symbol +-L = 32) takes g_s L2 / L3 activations to
    ~1e6 / ~1e12 -- beyond any fp16 representation.  The decode stays finite (saturated
    activations, never NaN), the overflow is counted, and x-hat stays in [0, 1]."""
    H, W = 128, 192
    c = lic.Codec(write_licw(HYPER, w), H, W)
    ys = _sym_plane(c, np.random.default_rng(6), 32)
    out = np.empty((1, 3, H, W), np.float32)
    c.range_count(reset=True)
    c.decode(ys, out)
    n = c.range_count()
    assert n > 0
    assert np.all(np.isfinite(out)) and out.min() >= 0 and out.max() <= 1
    ref = O.decode_frame(ys[0], w, True, O.pad_offsets(H, W, True)[2:], H, W)
    print(f"saturated plane: {n} activations saturated; x-hat agrees with the oracle on "
          f"{np.mean(np.abs(out[0] - ref) <= 1e-3):.3f} of the samples")
    c.close()


# ---------------------------------------------------------------- workspace
def test_bound_workspace_bit_identical(lic, w):
    import torch
    H, W, B = 136, 208, 2          # 3W % 16 == 0: the rebound row-halo g_a L1 and hi-only g_s L1 plans run
    c = lic.Codec(write_licw(HYPER, w), H, W, max_batch=B)
    fr = synth_frames_u8(B, H, W, seed=21)

    def run():
        ys = np.empty((B,) + c.y_shape, np.int8)
        yi = np.empty((B,) + c.y_shape, np.uint8)
        zs = np.empty((B,) + c.z_shape, np.int8)
        c.encode(fr, ys, yi, zs, u8=True)
        out = np.empty((B, H, W, 3), np.uint8)
        c.decode(ys, out, u8=True)
        return ys, yi, zs, out

    ref = run()
    nb = c.workspace_bytes()
    assert nb > 0 and c.workspace_bytes(1) < nb and c.workspace_bytes(B + 1) == 0
    ws = torch.empty(nb, dtype=torch.uint8, device="cuda")
    ws.fill_(0xAB)                                    # no reliance on zeroed memory
    assert c.bind_workspace(ws) == B
    got = run()
    for a, b in zip(ref, got):
        assert np.array_equal(a, b)
    # a one-frame block: max batch 1, per-frame results unchanged
    ws1 = torch.empty(c.workspace_bytes(1), dtype=torch.uint8, device="cuda")
    assert c.bind_workspace(ws1) == 1
    ys1 = np.empty((1,) + c.y_shape, np.int8)
    yi1 = np.empty((1,) + c.y_shape, np.uint8)
    zs1 = np.empty((1,) + c.z_shape, np.int8)
    c.encode(fr[1:2], ys1, yi1, zs1, u8=True)
    assert np.array_equal(ys1[0], ref[0][1]) and np.array_equal(yi1[0], ref[1][1])
    with pytest.raises(lic.LicError) as e:
        run()
    assert e.value.status == lic.LIC_ESHAPE
    with pytest.raises(lic.LicError) as e:
        c.bind_workspace(torch.empty(4096, dtype=torch.uint8, device="cuda"))
    assert e.value.status == lic.LIC_ENOSPACE
    host = np.empty(nb, np.uint8)
    with pytest.raises(lic.LicError) as e:
        c.bind_workspace(host, nb)
    assert e.value.status == lic.LIC_EINVAL
    c.close()
