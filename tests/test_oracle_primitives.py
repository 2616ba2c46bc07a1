"""Pins for the oracle primitives (-m "not gpu").

Each test pins the oracle to something other than itself: a SPEC.md worked
example, a closed form, an independent library routine (torch float64,
scipy), an algebraic identity, or brute force on tiny inputs.
"""
import math

import numpy as np
import pytest
import torch
import torch.nn.functional as F
from scipy.stats import norm

from oracle import oracle as O

RNG = np.random.default_rng(1234)


# ----------------------------------------------------------------- conv
def test_conv_spec_examples():
    # SPEC.md:49 1x1 kernel, weight 1, bias 0, stride 1 -> identity
    x = RNG.standard_normal((1, 5, 7)).astype(np.float32)
    out = O.conv2d(x, np.ones((1, 1, 1, 1), np.float32), np.zeros(1, np.float32), 1, 0)
    assert np.array_equal(out, x)
    # SPEC.md:50 4x4 ones * 2x2 ones, stride 2, padding 0 -> 2x2 of 4.0
    out = O.conv2d(np.ones((1, 4, 4), np.float32), np.ones((1, 1, 2, 2), np.float32),
                   np.zeros(1, np.float32), 2, 0)
    assert out.shape == (1, 2, 2) and np.all(out == 4.0)


@pytest.mark.parametrize("cin,cout,H,W,k,s", [(2, 3, 5, 5, 3, 1), (4, 2, 8, 8, 5, 2),
                                              (3, 4, 7, 6, 5, 2), (1, 1, 8, 8, 3, 1),
                                              (4, 4, 9, 8, 5, 2)])
def test_conv_vs_torch_float64(cin, cout, H, W, k, s):
    """agrees with an independent reference on <= 4 ch, <= 8x8."""
    p = k // 2
    x = RNG.standard_normal((cin, H, W)).astype(np.float32)
    w = RNG.standard_normal((cout, cin, k, k)).astype(np.float32)
    b = RNG.standard_normal(cout).astype(np.float32)
    ref = F.conv2d(torch.from_numpy(x).double()[None], torch.from_numpy(w).double(),
                   torch.from_numpy(b).double(), stride=s, padding=p)[0].float().numpy()
    out = O.conv2d(x, w, b, s, p)
    assert out.shape == ref.shape
    np.testing.assert_allclose(out, ref, rtol=1e-6, atol=1e-6)


def test_conv_full_layer_shape_vs_torch():
    """A g_a L2-shaped layer (N=128, 5x5/s2) at a small spatial size."""
    x = RNG.standard_normal((128, 12, 10)).astype(np.float32)
    w = (RNG.standard_normal((128, 128, 5, 5)) * 0.03).astype(np.float32)
    b = RNG.standard_normal(128).astype(np.float32)
    ref = F.conv2d(torch.from_numpy(x).double()[None], torch.from_numpy(w).double(),
                   torch.from_numpy(b).double(), stride=2, padding=2)[0].float().numpy()
    np.testing.assert_allclose(O.conv2d(x, w, b, 2, 2), ref, rtol=1e-6, atol=1e-6)


# ----------------------------------------------------------------- deconv
def test_deconv_spec_examples():
    # SPEC.md:59 stride 1, 1x1 unit kernel, padding 0 -> identity
    x = RNG.standard_normal((1, 4, 3)).astype(np.float32)
    out = O.deconv2d(x, np.ones((1, 1, 1, 1), np.float32), np.zeros(1, np.float32), 1, 0, 0)
    assert np.array_equal(out, x)
    # SPEC.md:60 1x1 input v, 2x2 ones, stride 2, padding 0 -> 2x2 of v
    out = O.deconv2d(np.full((1, 1, 1), 2.5, np.float32), np.ones((1, 1, 2, 2), np.float32),
                     np.zeros(1, np.float32), 2, 0, 0)
    assert out.shape == (1, 2, 2) and np.all(out == 2.5)


@pytest.mark.parametrize("cin,cout,H,W", [(2, 3, 3, 3), (4, 2, 4, 5), (3, 3, 1, 1), (4, 4, 6, 6)])
def test_deconv_vs_torch_float64(cin, cout, H, W):
    """5x5/s2/p2 with output_padding 1 vs torch conv_transpose2d.
    torch's ConvTranspose2d weight is in x out, ours out x in."""
    x = RNG.standard_normal((cin, H, W)).astype(np.float32)
    w = RNG.standard_normal((cout, cin, 5, 5)).astype(np.float32)
    b = RNG.standard_normal(cout).astype(np.float32)
    ref = F.conv_transpose2d(torch.from_numpy(x).double()[None],
                             torch.from_numpy(w).double().transpose(0, 1),
                             torch.from_numpy(b).double(), stride=2, padding=2,
                             output_padding=1)[0].float().numpy()
    out = O.deconv2d(x, w, b, 2, 2, 1)
    assert out.shape == (cout, 2 * H, 2 * W) == ref.shape
    np.testing.assert_allclose(out, ref, rtol=1e-6, atol=1e-6)


def test_conv_deconv_adjoint_identity():
    """<conv(x; W), u> == <x, deconv(u; W^T)> with zero bias (pins the deconv
    geometry convention against the conv's, independent of any library)."""
    cin, cout, H, W = 3, 4, 8, 6
    x = RNG.standard_normal((cin, H, W)).astype(np.float32)
    w = RNG.standard_normal((cout, cin, 5, 5)).astype(np.float32)
    u = RNG.standard_normal((cout, H // 2, W // 2)).astype(np.float32)
    cx = O.conv2d(x, w, np.zeros(cout, np.float32), 2, 2)
    dt = O.deconv2d(u, np.ascontiguousarray(w.transpose(1, 0, 2, 3)), np.zeros(cin, np.float32),
                    2, 2, 1)
    lhs = float(np.sum(cx.astype(np.float64) * u))
    rhs = float(np.sum(x.astype(np.float64) * dt))
    assert abs(lhs - rhs) <= 1e-4 * max(1.0, abs(lhs))


# ----------------------------------------------------------------- GDN
def _gdn_params(C, rng):
    beta = (1 + 0.1 * rng.random(C)).astype(np.float32)
    gamma = (0.1 * np.eye(C) + (0.1 / C) * rng.random((C, C))).astype(np.float32)
    return beta, gamma


def test_gdn_spec_examples():
    x = RNG.standard_normal((3, 4, 4)).astype(np.float32)
    one, zero = np.ones(3, np.float32), np.zeros((3, 3), np.float32)
    # SPEC.md:69 beta = 1, gamma = 0 -> identity (forward and inverse)
    assert np.array_equal(O.gdn(x, one, zero), x)
    assert np.array_equal(O.gdn(x, one, zero, inverse=True), x)
    # SPEC.md:70 single channel x=3, beta=7, gamma=1 -> 3/sqrt(16) = 0.75
    out = O.gdn(np.full((1, 1, 1), 3.0, np.float32), np.array([7.0], np.float32),
                np.array([[1.0]], np.float32))
    assert out[0, 0, 0] == np.float32(0.75)
    # the scalar IGDN of 0.75 is 0.75*sqrt(7+0.5625) = 2.0625, not 3
    inv = O.gdn(out, np.array([7.0], np.float32), np.array([[1.0]], np.float32), inverse=True)
    assert inv[0, 0, 0] == np.float32(2.0625)


def test_gdn_gamma_zero_roundtrip():
    """c12 (i): gamma = 0 -> IGDN(GDN(x)) = x (to fp32 double-rounding)."""
    C = 8
    x = RNG.standard_normal((C, 5, 5)).astype(np.float32)
    beta = (1 + RNG.random(C)).astype(np.float32)
    g0 = np.zeros((C, C), np.float32)
    np.testing.assert_allclose(O.gdn(O.gdn(x, beta, g0), beta, g0, inverse=True), x, rtol=3e-7)


def test_gdn_fixed_point_inverse():
    """c12 (ii)/(iii): x = y * sqrt(beta + gamma x^2) where y = GDN(x); the
    fixed-point iteration x_{t+1} = y * sqrt(beta + gamma x_t^2) recovers x.
    A transposed gamma or a dropped beta in the oracle breaks this."""
    C = 16
    beta, gamma = _gdn_params(C, RNG)
    gamma = gamma + 0.02 * RNG.random((C, C)).astype(np.float32)  # asymmetric
    x = RNG.standard_normal((C, 3, 3)).astype(np.float32)
    y = O.gdn(x, beta, gamma).astype(np.float64)
    X = x.reshape(C, -1).astype(np.float64)
    Y = y.reshape(C, -1)
    g, b = gamma.astype(np.float64), beta.astype(np.float64)[:, None]
    # (iii) identity on the true x
    np.testing.assert_allclose(Y * np.sqrt(b + g @ X ** 2), X, rtol=1e-6, atol=1e-6)
    # (ii) fixed point from y
    xt = Y.copy()
    for _ in range(200):
        xt = Y * np.sqrt(b + g @ xt ** 2)
    np.testing.assert_allclose(xt, X, rtol=1e-5, atol=1e-5)


def test_gdn_vs_torch_composition():
    C = 32
    beta, gamma = _gdn_params(C, RNG)
    x = (RNG.standard_normal((C, 6, 7)) * 2).astype(np.float32)
    xt = torch.from_numpy(x).double()
    n = torch.from_numpy(beta).double()[:, None, None] + torch.einsum(
        "ij,jhw->ihw", torch.from_numpy(gamma).double(), xt * xt)
    np.testing.assert_allclose(O.gdn(x, beta, gamma), (xt / n.sqrt()).float().numpy(), rtol=1e-6)
    np.testing.assert_allclose(O.gdn(x, beta, gamma, inverse=True), (xt * n.sqrt()).float().numpy(),
                               rtol=1e-6)


def test_onedn_spec_examples():
    x = RNG.standard_normal((2, 3, 3)).astype(np.float32)
    assert np.array_equal(O.onedn(x, np.ones(2, np.float32), np.zeros((2, 2), np.float32)), x)
    # SPEC.md:80 x=3, beta=1, gamma=1 -> 3/(1+3) = 0.75
    out = O.onedn(np.full((1, 1, 1), 3.0, np.float32), np.ones(1, np.float32),
                  np.ones((1, 1), np.float32))
    assert out[0, 0, 0] == np.float32(0.75)
    # sign/abs pin: x = -3 -> -0.75
    out = O.onedn(np.full((1, 1, 1), -3.0, np.float32), np.ones(1, np.float32),
                  np.ones((1, 1), np.float32))
    assert out[0, 0, 0] == np.float32(-0.75)


# ----------------------------------------------------------------- quantise
def test_quantize_spec_examples():
    # SPEC.md:198 y = 1.4, mu = 0.25 -> symbol 1, yhat = 1.25
    s, yh, ns = O.quantize(np.full((1, 1, 1), 1.4, np.float32), np.array([0.25], np.float32), 32)
    assert s[0, 0, 0] == 1 and yh[0, 0, 0] == np.float32(1.25) and ns == 0
    # SPEC.md:197 mu = 0 and integer-valued y -> fixed point
    y = RNG.integers(-32, 33, size=(3, 4, 4)).astype(np.float32)
    s, yh, ns = O.quantize(y, np.zeros(3, np.float32), 32)
    assert np.array_equal(yh, y) and np.array_equal(s.astype(np.float32), y) and ns == 0


def test_quantize_ties_and_clamp():
    """c4: half away from zero (not half-even); c6: clamp to +-L with a count."""
    y = np.array([2.5, -2.5, 0.5, -0.5, 1.5, 32.5, -32.5, 31.49, 100.0], np.float32).reshape(1, 1, -1)
    s, yh, ns = O.quantize(y, None, 32)
    assert s.ravel().tolist() == [3, -3, 1, -1, 2, 32, -32, 31, 32]
    assert ns == 3


def test_quantize_rounding_bound():
    """dequantize(quantize(y)) within 0.5 of y when unsaturated."""
    y = (RNG.standard_normal((4, 8, 8)) * 5).astype(np.float32)
    mu = RNG.uniform(-0.25, 0.25, 4).astype(np.float32)
    s, yh, ns = O.quantize(y, mu, 32)
    assert ns == 0
    assert np.max(np.abs(yh - y)) <= 0.5 + 1e-6
    assert np.array_equal(O.dequantize(s, mu), yh)


# ----------------------------------------------------------------- scale index
def test_scale_index_spec_examples():
    t = np.array([0.11, 0.22, 0.44], np.float32)
    assert O.scale_index(np.array([0.11], np.float32), t)[0] == 0
    assert O.scale_index(np.array([0.30], np.float32), t)[0] == 2
    assert O.scale_index(np.array([1e6], np.float32), t)[0] == 2      # SPEC.md:189 (last)
    assert O.scale_index(np.array([0.0, -1.0], np.float32), t).tolist() == [0, 0]  # lower bound


def test_scale_index_vs_searchsorted():
    """Brute force against numpy.searchsorted(side='left') = #{table < s'}."""
    from lic_synth import scale_table
    t = scale_table()
    sig = np.concatenate([RNG.uniform(0, 300, 20000).astype(np.float32), t, t * 1.0000001,
                          np.nextafter(t, 0)]).astype(np.float32)
    ref = np.minimum(np.searchsorted(t[:-1], np.maximum(sig, np.float32(0.11)), side="left"), 63)
    assert np.array_equal(O.scale_index(sig, t), ref.astype(np.uint8))


# ----------------------------------------------------------------- CDF
def _check_row(c, L):
    f = np.diff(c.astype(np.int64))
    assert c[0] == 0 and c[-1] == 65536 and len(c) == 2 * L + 2
    assert np.all(f >= 1)
    assert np.array_equal(f, f[::-1])              # zero-mean rows are symmetric
    return f


def test_cdf_spec_examples():
    # SPEC.md:169 sigma = 0.05, L = 8 -> centre >= 2^16 - 2L; c8 rule gives exactly 65520
    f = _check_row(O.cdf_row(0.05, 8), 8)
    assert f[8] == 65520
    for s in np.linspace(0.11, 256, 40):
        _check_row(O.cdf_row(float(s), 32), 32)


def test_cdf_vs_scipy_phi():
    """probabilities match a direct Phi-difference oracle within
    quantisation (+-1 frequency unit off-centre); scipy's norm is independent."""
    from lic_synth import scale_table
    L = 32
    for s in list(scale_table()) + [0.5, 0.77, 1.0, 1.5]:
        s = float(np.float32(s))
        f = _check_row(O.cdf_row(s, L), L)
        k = np.arange(-L, L + 1)
        p = norm.cdf((k + 0.5) / s) - norm.cdf((k - 0.5) / s)
        p[0] = norm.cdf((-L + 0.5) / s)
        p[-1] = p[0]
        d = f - p * 65536
        off = np.abs(k) != 0
        assert np.max(np.abs(d[off])) <= 1.0 + 1e-6
        assert abs(d[L]) <= 2 * L + 1


def test_cdf_entropy_increases_with_sigma():
    """the row for the largest sigma is flatter (higher entropy) than
    the row for the smallest.  Strict monotonicity holds only while the tail
    folded into +-L is negligible (sigma <= 8 here): with L = 32 the folded edge
    bins dominate for sigma >> L and the entropy falls again (R9)."""
    from lic_synth import scale_table
    t = scale_table()
    H = []
    for s in t:
        f = np.diff(O.cdf_row(float(s), 32).astype(np.float64)) / 65536
        H.append(-np.sum(f * np.log2(f)))
    H = np.array(H)
    assert H[-1] > H[0]
    assert np.all(np.diff(H[t <= 8.0]) > 0)


# ----------------------------------------------------------------- rANS
@pytest.mark.parametrize("cdf,sym,hexstr", [
    ([0, 32768, 65536], [0, 1], "02010000"),
    ([0, 32768, 65536], [], "00800000"),
    ([0, 1, 65536], [0], "008000000000"),
    ([0, 100, 40000, 65536], [2, 1, 0, 1, 2, 2, 1, 1], "009dc5b89250"),
])
def test_rans_known_answers(cdf, sym, hexstr):
    """Hand-derivable known answers.  E.g. the first:
    x=2^23; s=1 (start 32768, freq 32768) -> x = 2^24 + 2^15; s=0 -> x = 2^25 + 2^16
    = 0x02010000, flushed big-endian."""
    c = np.array(cdf, np.uint32)[None]
    b = O.rans_encode(np.array(sym, np.int8), np.zeros(len(sym)), c, sym_min=0)
    assert b.hex() == hexstr
    assert O.rans_decode(b, np.zeros(len(sym)), c, sym_min=0).tolist() == list(sym)


def test_rans_skewed_1000():
    """1000 x A with P(A) = 64881/65536: cross-entropy 14.5 bits;
    the coder emits 5 bytes (SPEC.md:149's 11-27 bytes is wrong)."""
    c = np.array([0, 64881, 65536], np.uint32)[None]
    b = O.rans_encode(np.zeros(1000, np.int8), np.zeros(1000), c, sym_min=0)
    bits = -1000 * math.log2(64881 / 65536)
    assert len(b) == 5 and len(b) <= math.ceil(bits / 8) + 16


def test_rans_million_roundtrip_and_efficiency():
    """SPEC.md:598 acceptance #1: 10^6 symbols across 192 rows round-trip exactly;
    bits <= cross-entropy + 128."""
    L = 32
    sig = RNG.uniform(0.2, 8.0, 192)
    cdf = O.cdf_table(sig, L)
    n = 1_000_000
    rows = RNG.integers(0, 192, n).astype(np.int32)
    # draw symbols from the rows' own distributions
    u = RNG.integers(0, 65536, n)
    sym = np.empty(n, np.int8)
    for r in range(192):
        m = rows == r
        sym[m] = (np.searchsorted(cdf[r], u[m], side="right") - 1 - L).astype(np.int8)
    b = O.rans_encode(sym, rows, cdf)
    assert np.array_equal(O.rans_decode(b, rows, cdf), sym)
    f = np.diff(cdf.astype(np.float64), axis=1) / 65536
    xent = -np.sum(np.log2(f[rows, sym.astype(np.int64) + L]))
    assert 8 * len(b) <= xent + 128


def test_rans_corrupt_streams():
    """SPEC.md:160 truncated byte string -> explicit corrupt-stream error."""
    L = 32
    cdf = O.cdf_table([1.0, 3.0], L)
    rows = RNG.integers(0, 2, 5000)
    sym = np.clip(np.round(RNG.standard_normal(5000) * 2), -L, L).astype(np.int8)
    b = O.rans_encode(sym, rows, cdf)
    for cut in (1, 2, len(b) // 2, len(b) - 4):
        with pytest.raises(O.CorruptStream):
            O.rans_decode(b[:-cut], rows, cdf)
    with pytest.raises(O.CorruptStream):
        O.rans_decode(b + b"\x00", rows, cdf)
    with pytest.raises(O.CorruptStream):
        O.rans_decode(b"", rows, cdf)


def test_rans_slabs_framing_pins():
    """DESIGN.md R21: K = 1 is the plain string (known answer);
    K > 1 = big-endian u32 lengths + independent strings of channel slabs
    [floor(kC/K), floor((k+1)C/K)).  Pinned without the slab code: each substring equals the
    plain coder run on that slab alone with its own rows (so a dropped row offset or a wrong
    slab boundary fails), and the framing sizes add up."""
    rng = np.random.default_rng(11)
    L = 32
    C, H, W = 7, 3, 5
    sig = rng.uniform(0.5, 2.0, C)
    cdf = O.cdf_table(sig, L)
    sym = np.clip(np.round(rng.standard_normal((C, H, W)) * 2), -L, L).astype(np.int8)
    assert O.rans_encode_slabs(sym, None, cdf, 1) == O.rans_encode(sym, O.channel_rows(sym.shape), cdf)
    b = O.rans_encode_slabs(sym, None, cdf, 3)
    lens = [int.from_bytes(b[4 * k:4 * k + 4], "big") for k in range(3)]
    assert 12 + sum(lens) == len(b)
    bounds = [(0, 2), (2, 4), (4, 7)]            # floor(k*7/3): 0, 2, 4, 7
    pos = 12
    for (c0, c1_), n in zip(bounds, lens):
        # the slab coded alone with a table holding only its own channels' rows
        sub_cdf = O.cdf_table(sig[c0:c1_], L)
        plain = O.rans_encode(sym[c0:c1_], O.channel_rows(sym[c0:c1_].shape), sub_cdf)
        assert b[pos:pos + n] == plain
        pos += n
    assert np.array_equal(O.rans_decode_slabs(b, sym.shape, None, cdf, 3), sym)
    with pytest.raises(O.CorruptStream):
        O.rans_decode_slabs(b[:-1], sym.shape, None, cdf, 3)


def test_onedn_gamma_zero_roundtrip_and_fixed_point():
    """1DN: gamma = 0 -> inverse(forward(x)) = x; in general
    x = y * (beta + gamma |x|) for y = 1DN(x), and the fixed-point iteration
    x_{t+1} = y * (beta + gamma |x_t|) recovers x (a transposed gamma, x^2 in place of |x|
    or a dropped beta breaks one of these)."""
    C = 12
    rng = np.random.default_rng(5)
    x = rng.standard_normal((C, 4, 4)).astype(np.float32)
    beta = (1 + rng.random(C)).astype(np.float32)
    g0 = np.zeros((C, C), np.float32)
    np.testing.assert_allclose(O.onedn(O.onedn(x, beta, g0), beta, g0, inverse=True), x, rtol=3e-7)
    beta, gamma = _gdn_params(C, rng)
    gamma = gamma + 0.02 * rng.random((C, C)).astype(np.float32)
    y = O.onedn(x, beta, gamma).astype(np.float64)
    X, Y = x.reshape(C, -1).astype(np.float64), y.reshape(C, -1)
    g, b = gamma.astype(np.float64), beta.astype(np.float64)[:, None]
    np.testing.assert_allclose(Y * (b + g @ np.abs(X)), X, rtol=1e-6, atol=1e-6)
    xt = Y.copy()
    for _ in range(300):
        xt = Y * (b + g @ np.abs(xt))
    np.testing.assert_allclose(xt, X, rtol=1e-5, atol=1e-5)
    # the inverse is the multiply form on the same norm
    inv = O.onedn(x, beta, gamma, inverse=True).astype(np.float64).reshape(C, -1)
    np.testing.assert_allclose(inv, X * (b + g @ np.abs(X)), rtol=1e-6)
