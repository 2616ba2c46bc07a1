"""Whole-network oracle pins (-m "not gpu").

The transforms are pinned against an independent torch-float64 composition of
the same layer list, built here from torch's own conv /
conv_transpose; the codec against latent fidelity (SPEC.md:268, :279, :289,
:314) and determinism.
"""
import numpy as np
import pytest
import torch
import torch.nn.functional as F

from lic_synth import ModelSpec, generate_weights, synth_frame_u8
from oracle import oracle as O

HYPER = ModelSpec(kind=1, N=128, M=192)
FACT = ModelSpec(kind=0, N=128, M=192)


def _t(a):
    return torch.from_numpy(np.ascontiguousarray(a)).double()


def _gdn64(x, beta, gamma, inverse):
    n = _t(beta)[:, None, None] + torch.einsum("ij,jhw->ihw", _t(gamma), x * x)
    return x * n.sqrt() if inverse else x / n.sqrt()


def torch_ga(x, w):
    h = _t(x)
    for i in (1, 2, 3):
        h = F.conv2d(h[None], _t(w[f"ga{i}.w"]), _t(w[f"ga{i}.b"]), stride=2, padding=2)[0]
        h = _gdn64(h, w[f"ga{i}.beta"], w[f"ga{i}.gamma"], False)
    return F.conv2d(h[None], _t(w["ga4.w"]), _t(w["ga4.b"]), stride=2, padding=2)[0]


def torch_gs(y, w):
    h = _t(y)
    for i in (1, 2, 3):
        h = F.conv_transpose2d(h[None], _t(w[f"gs{i}.w"]).transpose(0, 1), _t(w[f"gs{i}.b"]),
                               stride=2, padding=2, output_padding=1)[0]
        h = _gdn64(h, w[f"gs{i}.beta"], w[f"gs{i}.gamma"], True)
    return F.conv_transpose2d(h[None], _t(w["gs4.w"]).transpose(0, 1), _t(w["gs4.b"]),
                              stride=2, padding=2, output_padding=1)[0]


def torch_ha(y, w):
    h = F.relu(F.conv2d(_t(np.abs(y))[None], _t(w["ha1.w"]), _t(w["ha1.b"]), padding=1))
    h = F.relu(F.conv2d(h, _t(w["ha2.w"]), _t(w["ha2.b"]), stride=2, padding=2))
    return F.conv2d(h, _t(w["ha3.w"]), _t(w["ha3.b"]), stride=2, padding=2)[0]


def torch_hs(z, w):
    h = F.relu(F.conv_transpose2d(_t(z)[None], _t(w["hs1.w"]).transpose(0, 1), _t(w["hs1.b"]),
                                  stride=2, padding=2, output_padding=1))
    h = F.relu(F.conv_transpose2d(h, _t(w["hs2.w"]).transpose(0, 1), _t(w["hs2.b"]),
                                  stride=2, padding=2, output_padding=1))
    return F.relu(F.conv2d(h, _t(w["hs3.w"]), _t(w["hs3.b"]), padding=1))[0]


@pytest.fixture(scope="module")
def hyper_case():
    w = generate_weights(HYPER, seed=0)
    frame = synth_frame_u8(128, 128, seed=3, t=0)
    x, crop = O.ingest_u8(frame, hyper=True)
    return w, x, crop


def test_transforms_vs_torch_float64(hyper_case):
    """Each transform on the same fp32 input: oracle (fp64 per layer, fp32 between
    layers) vs torch float64 end to end.  The only difference is the fp32 rounding
    between layers, so agreement to ~1e-5 pins every layer's indexing and math."""
    w, x, _ = hyper_case
    y = O.g_a(x, w)
    np.testing.assert_allclose(y, torch_ga(x, w).numpy(), atol=2e-5, rtol=0)
    z = O.h_a(y, w)
    np.testing.assert_allclose(z, torch_ha(y, w).numpy(), atol=2e-5, rtol=0)
    zs, zhat, _ = O.quantize(z, w["mu_z"], 32)
    s = O.h_s(zhat, w)
    np.testing.assert_allclose(s, torch_hs(zhat, w).numpy(), atol=2e-5, rtol=1e-6)
    ys, yhat, _ = O.quantize(y, None, 32)
    xs = O.g_s(yhat, w)
    np.testing.assert_allclose(xs, torch_gs(yhat, w).numpy(), atol=2e-5, rtol=0)


def _onedn64(x, beta, gamma, inverse):
    n = _t(beta)[:, None, None] + torch.einsum("ij,jhw->ihw", _t(gamma), x.abs())
    return x * n if inverse else x / n


def test_onedn_transforms_vs_torch_float64(hyper_case):
    """1DN variant (the paper's implementation C): oracle g_a / g_s with
    act = 1 against a torch float64 composition of conv / conv_transpose and the 1DN
    formula."""
    w, x, _ = hyper_case
    h = _t(x)
    for i in (1, 2, 3):
        h = F.conv2d(h[None], _t(w[f"ga{i}.w"]), _t(w[f"ga{i}.b"]), stride=2, padding=2)[0]
        h = _onedn64(h, w[f"ga{i}.beta"], w[f"ga{i}.gamma"], False)
    y_ref = F.conv2d(h[None], _t(w["ga4.w"]), _t(w["ga4.b"]), stride=2, padding=2)[0].numpy()
    y = O.g_a(x, w, act=1)
    np.testing.assert_allclose(y, y_ref, atol=2e-5, rtol=0)
    assert np.abs(y - O.g_a(x, w)).max() > 1e-2                     # really a different activation
    yh = np.round(y).astype(np.float32)
    g = _t(yh)
    for i in (1, 2, 3):
        g = F.conv_transpose2d(g[None], _t(w[f"gs{i}.w"]).transpose(0, 1), _t(w[f"gs{i}.b"]),
                               stride=2, padding=2, output_padding=1)[0]
        g = _onedn64(g, w[f"gs{i}.beta"], w[f"gs{i}.gamma"], True)
    xr = F.conv_transpose2d(g[None], _t(w["gs4.w"]).transpose(0, 1), _t(w["gs4.b"]),
                            stride=2, padding=2, output_padding=1)[0].numpy()
    np.testing.assert_allclose(O.g_s(yh, w, act=1), xr, atol=2e-5, rtol=1e-5)


def test_latents_are_not_degenerate(hyper_case):
    """SURVEY.md finding 2 / c15: the init must exercise the coder (non-zero
    symbols, several CDF indexes), else parity passes vacuously."""
    w, x, _ = hyper_case
    p = O.encode_planes(x, w, True, 32)
    assert 0.1 < np.mean(p["y_sym"] != 0) < 0.6
    assert len(np.unique(p["y_idx"])) >= 5
    assert p["n_sat"] == 0


def test_hyper_codec_latent_fidelity_and_determinism(hyper_case):
    w, x, crop = hyper_case
    t = O.build_tables(w, True, 32)
    p = O.encode_planes(x, w, True, 32)
    yb, zb = O.code_planes(p, t, True)
    p2 = O.encode_planes(x, w, True, 32)
    assert O.code_planes(p2, t, True) == (yb, zb)
    xh, ys = O.decode_strings(yb, zb, w, t, True, p["y_sym"].shape, p["z_sym"].shape, crop,
                              128, 128)
    assert np.array_equal(ys, p["y_sym"])
    assert np.array_equal(O.hyper_indexes(p["z_sym"], w), p["y_idx"])     # GPU1 == encoder
    assert xh.shape == (3, 128, 128) and xh.min() >= 0 and xh.max() <= 1


def test_factorized_codec_latent_fidelity():
    w = generate_weights(FACT, seed=0)
    frame = synth_frame_u8(64, 64, seed=1, t=0)
    x, crop = O.ingest_u8(frame, hyper=False)
    t = O.build_tables(w, False, 32)
    p = O.encode_planes(x, w, False, 32)
    yb, _ = O.code_planes(p, t, False)
    xh, ys = O.decode_strings(yb, None, w, t, False, p["y_sym"].shape, None, crop, 64, 64)
    assert np.array_equal(ys, p["y_sym"])
    assert np.array_equal(O.dequantize(ys, w["mu_y"]), p["yhat"])
    np.testing.assert_allclose(xh, np.clip(torch_gs(p["yhat"], w).numpy(), 0, 1)[:, :64, :64],
                               atol=2e-5)


def test_padding_geometry():
    """720 -> 768 and 1080 -> 1088 (hyper 64, fact 16), centred."""
    assert O.pad_offsets(720, 1280, True) == (768, 1280, 24, 0)
    assert O.pad_offsets(1080, 1920, True) == (1088, 1920, 4, 0)
    assert O.pad_offsets(512, 768, False) == (512, 768, 0, 0)
    assert O.pad_offsets(1080, 1920, False) == (1088, 1920, 4, 0)
    f = synth_frame_u8(40, 50, seed=0)
    x, (top, left) = O.ingest_u8(f, hyper=False)
    assert x.shape == (3, 48, 64) and (top, left) == (4, 7)
    assert np.all(x[:, :top] == 0) and np.all(x[:, :, :left] == 0)
    assert x[0, top, left] == np.float32(f[0, 0, 0]) / np.float32(255)
