"""rans64 + bypass escape coder (R23), -m "not gpu".

Oracle pins (oracle/rans64.py against values worked out by hand from the definitions, the
quantiser's rounding rule, the ideal code length) and the product coder (lic_rans64_*,
lic_cdf_quantize, lic_cdf64_gaussian through the C ABI) bit-exact against the oracle.
"""
import math
import struct

import numpy as np
import pytest

from oracle import rans64 as O
from paper_2208_01641_b200 import lic

# one row: symbols 0 (freq 32768), 1 (freq 32767), escape (freq 1)
CDF1 = np.array([[0, 32768, 65535, 65536]], np.uint32)
SIZES1, OFFS1 = [4], [0]


# ------------------------------------------------------------------ oracle pins (by hand)

def test_oracle_single_symbol_states_by_hand():
    # x0 = 2^31.  Put(start 0, freq 2^15): x < x_max = 2^62, x = (2^31 / 2^15) << 16 = 2^32
    assert O.rans64_encode([0], [0], CDF1, SIZES1, OFFS1) == struct.pack("<II", 0, 1)
    # Put(start 32768, freq 32767): 2^31 = 65538 * 32767 + 2 -> x = 65538 << 16 | (2 + 32768)
    x = (65538 << 16) + 2 + 32768
    assert x == 0x1_0002_8002
    assert O.rans64_encode([1], [0], CDF1, SIZES1, OFFS1) == struct.pack("<II", x & 0xFFFFFFFF, x >> 32)


def test_oracle_escape_by_hand():
    # s = 5 >= v_max = 2: raw = 2 (5 - 2) = 6, one 4-bit chunk.  Pushes: escape (65535, 1),
    # count 1, chunk 6; coded in reverse: x = 2^31 << 4 | 6, then << 4 | 1, then the escape
    # x = x << 16 | 65535 (freq 1: x / 1 = x, no renormalisation below 2^47)
    x = (((1 << 31) << 4 | 6) << 4 | 1)
    x = (x << 16) + 65535
    assert x == (1 << 55) + 6422527
    assert O.rans64_encode([5], [0], CDF1, SIZES1, OFFS1) == struct.pack("<II", x & 0xFFFFFFFF, x >> 32)
    # negative values: raw = -2v - 1 (odd), v = -1 -> raw 1
    x = (((1 << 31) << 4 | 1) << 4 | 1)
    x = (x << 16) + 65535
    assert O.rans64_encode([-1], [0], CDF1, SIZES1, OFFS1) == struct.pack("<II", x & 0xFFFFFFFF, x >> 32)


def test_oracle_escape_count_chunks():
    # a raw value with 16 chunks (>= 15) sends its count as 15 then 1
    syms = O.symbol_list([2 + (1 << 62)], [0], CDF1, SIZES1, OFFS1)   # raw = 2^63: 16 chunks
    assert syms[0] == (65535, 1, False)
    assert [s[0] for s in syms[1:3]] == [15, 1]
    assert len(syms) == 3 + 16 and syms[-1][0] == 8


def test_quantizer_by_hand():
    assert O.pmf_to_quantized_cdf([0.5, 0.25, 0.25]).tolist() == [0, 32768, 49152, 65536]
    # a zero frequency takes one slot from the smallest frequency > 1
    assert O.pmf_to_quantized_cdf([1.0, 0.0]).tolist() == [0, 65535, 65536]
    assert O.pmf_to_quantized_cdf([0.0, 1.0]).tolist() == [0, 1, 65536]
    # p * 2^16 = 1.5 and 65534.5 round half away from zero to 2 and 65535 (total 65537,
    # rescaled to 1 and 65533, last pinned to 2^16); half-to-even would give [0, 2, 65536]
    p = 1.5 / 65536
    assert O.pmf_to_quantized_cdf([p, 1.0 - p]).tolist() == [0, 1, 65536]


def test_oracle_round_trip_and_ideal_length():
    rng = np.random.default_rng(0)
    pmf = rng.random(24)
    pmf = list(pmf / pmf.sum() * 0.999) + [0.001]
    cdf = O.pmf_to_quantized_cdf(pmf)[None]
    n = 6000
    sym = rng.integers(-3, 27, n) - 2           # values outside [0, 24) are escapes
    idx = np.zeros(n, int)
    sizes, offs = [cdf.shape[1]], [-2]
    b = O.rans64_encode(sym, idx, cdf, sizes, offs)
    assert len(b) % 4 == 0
    assert (O.rans64_decode(b, idx, cdf, sizes, offs) == sym).all()
    ideal = O.ideal_bits(sym, idx, cdf, sizes, offs)
    # rANS costs the information content up to the flushed state and the last partial word
    assert ideal - 32 <= 8 * len(b) <= ideal + 96


def test_oracle_gaussian_multiplier_and_widths():
    cdfs, sizes, offs = O.gaussian_tables([1.0, 0.11, 10.0])
    m = -O_ppf(5e-10)
    assert abs(m - 6.1094102) < 1e-6
    assert offs.tolist() == [-math.ceil(1.0 * m), -math.ceil(np.float32(0.11) * m), -math.ceil(10.0 * m)]
    assert sizes.tolist() == [2 * -o + 3 for o in offs]
    for r in range(3):
        f = np.diff(cdfs[r, : sizes[r]].astype(np.int64))
        assert f.min() >= 1 and cdfs[r, sizes[r] - 1] == 65536
    # scale 1: the centre bin holds P(|X| < 1/2) = erf(1/(2 sqrt 2)) of the mass
    c = -offs[0]
    f0 = int(cdfs[0, c + 1]) - int(cdfs[0, c])
    assert abs(f0 / 65536 - math.erf(0.5 / math.sqrt(2))) < 2e-4


def O_ppf(q):
    from statistics import NormalDist
    return NormalDist().inv_cdf(q)


# ------------------------------------------------------------------ product vs oracle

def test_product_hand_pins():
    T = lic.Rans64Tables(CDF1, SIZES1, OFFS1)
    for v in (0, 1, 5, -1):
        assert T.encode([v], [0]) == O.rans64_encode([v], [0], CDF1, SIZES1, OFFS1)
    assert lic.cdf_quantize([1.5 / 65536, 1.0 - 1.5 / 65536]).tolist() == [0, 1, 65536]


@pytest.mark.parametrize("seed", [0, 1, 2, 3])
def test_quantizer_matches_oracle(seed):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(2, 300))
    pmf = rng.random(n) ** 6                     # many tiny masses: exercises the stealing
    pmf[rng.integers(0, n, n // 4)] = 0.0
    pmf = (pmf / pmf.sum()).astype(np.float32)
    assert (lic.cdf_quantize(pmf) == O.pmf_to_quantized_cdf(pmf)).all()


def _scales():
    # the codec's scale table shape: 64 log-spaced scales
    return np.exp(np.linspace(np.log(0.11), np.log(256.0), 64)).astype(np.float32)


def test_gaussian_tables_match_oracle():
    G = lic.Rans64Tables.gaussian(_scales())
    c, s, o = O.gaussian_tables(_scales(), stride=G.cdfs.shape[1])
    assert (G.cdfs == c).all() and (G.sizes == s).all() and (G.offsets == o).all()


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_codec_shaped_stream_bit_exact(seed):
    """Indexed Gaussian rows, values drawn wider than the tables (escapes at every scale),
    plus int32 extremes."""
    G = lic.Rans64Tables.gaussian(_scales())
    rng = np.random.default_rng(seed)
    n = 5000
    idx = rng.integers(0, 64, n)
    sym = np.round(rng.standard_t(2, n) * _scales()[idx]).clip(-2**31, 2**31 - 1).astype(np.int32)
    sym[:4] = [2**31 - 1, -2**31, 0, -1]
    b = G.encode(sym, idx)
    assert b == O.rans64_encode(sym, idx, G.cdfs, G.sizes, G.offsets)
    assert (G.decode(b, idx) == sym).all()
    assert (O.rans64_decode(b, idx, G.cdfs, G.sizes, G.offsets) == sym).all()


def test_empty_and_large_round_trip():
    G = lic.Rans64Tables.gaussian(_scales())
    assert G.encode([], []) == struct.pack("<II", 1 << 31, 0)
    assert G.decode(G.encode([], []), []).size == 0
    rng = np.random.default_rng(7)
    n = 1 << 20
    idx = rng.integers(0, 64, n)
    sym = np.round(rng.normal(0, 1, n) * _scales()[idx]).astype(np.int32)
    b = G.encode(sym, idx)
    assert (G.decode(b, idx) == sym).all()


def test_corrupt_streams_fail_cleanly():
    G = lic.Rans64Tables.gaussian(_scales())
    rng = np.random.default_rng(3)
    n = 3000
    idx = rng.integers(0, 64, n)
    sym = np.round(rng.normal(0, 2, n) * _scales()[idx]).astype(np.int32)
    b = G.encode(sym, idx)
    for cut in (0, 4, 7, len(b) - 4, len(b) - 1):
        with pytest.raises(lic.CorruptStream):
            G.decode(b[:cut], idx)
    with pytest.raises(lic.CorruptStream):
        G.decode(b + b"\0\0\0\0", idx)               # words left over
    for k in range(40):                              # flipped bits: an error or wrong output, no crash
        bb = bytearray(b)
        bb[int(rng.integers(0, len(b)))] ^= 1 << int(rng.integers(0, 8))
        try:
            out = G.decode(bytes(bb), idx)
            assert out.shape == sym.shape
        except lic.CorruptStream:
            pass


def test_invalid_tables_and_rows():
    bad = np.array([[0, 40000, 30000, 65536]], np.uint32)          # not increasing
    with pytest.raises(lic.LicError):
        lic.Rans64Tables(bad, [4], [0]).encode([0], [0])
    with pytest.raises(lic.LicError):
        lic.Rans64Tables(CDF1, [4], [0]).encode([0], [1])            # row out of range
    with pytest.raises(lic.LicError):
        lic.cdf_quantize([0.0, 0.0])


def test_codec_planes_with_rans64():
    """The hyperprior's y plane (oracle encode, 128 x 128 frame) coded with rows = its CDF
    indexes and CompressAI-style tables on the codec's own scale table: bit-exact with the
    oracle, lossless, and within a few percent of the clamped 32-bit rANS string."""
    from lic_synth import ModelSpec, generate_weights, synth_frame_u8
    from oracle import oracle as OR

    w = generate_weights(ModelSpec(kind=1, N=128, M=192), seed=0)
    x, _ = OR.ingest_u8(synth_frame_u8(128, 128, seed=3, t=0), hyper=True)
    p = OR.encode_planes(x, w, True, 32)
    sym, idx = p["y_sym"].astype(np.int32), p["y_idx"].astype(np.int32)
    G = lic.Rans64Tables.gaussian(w["scale_table"])
    b = G.encode(sym, idx)
    assert b == O.rans64_encode(sym.ravel(), idx.ravel(), G.cdfs, G.sizes, G.offsets)
    assert (G.decode(b, idx).reshape(sym.shape) == sym).all()
    b32 = OR.rans_encode(p["y_sym"], p["y_idx"], OR.build_tables(w, True, 32).gauss)
    assert abs(len(b) - len(b32)) <= 0.05 * len(b32) + 16
