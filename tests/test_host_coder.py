"""Product host coder (liblic.so) vs the oracle, bit-exact (-m "not gpu").

SURVEY.md §8(c) c19 (i): rANS(planes) == oracle rANS(planes) byte-for-byte, always;
CDF tables identical to the oracle's.
"""
import numpy as np
import pytest

from lic_synth import ModelSpec, generate_weights, scale_table, write_licw, read_licw_blocks
from oracle import oracle as O

RNG = np.random.default_rng(7)


@pytest.fixture(scope="module")
def lic():
    from paper_2208_01641_b200 import build
    build.build()
    from paper_2208_01641_b200 import lic as L
    return L


def test_cdf_tables_bit_exact(lic):
    t = scale_table()
    sig = np.concatenate([t, RNG.uniform(0.05, 300, 200).astype(np.float32),
                          np.array([0.11, 0.5, 1.0, 1.5], np.float32)])
    for L in (8, 32):
        assert np.array_equal(lic.cdf_build(sig, L), O.cdf_table(sig, L))


def test_rans_kats(lic):
    c = np.array([[0, 100, 40000, 65536]], np.uint32)
    b = lic.rans_encode(np.array([2, 1, 0, 1, 2, 2, 1, 1], np.int8), c, rows=np.zeros(8, np.uint8), sym_min=0)
    assert b.hex() == "009dc5b89250"
    c = np.array([[0, 32768, 65536]], np.uint32)
    assert lic.rans_encode(np.zeros((0,), np.int8), c, rows=np.zeros(0, np.uint8), sym_min=0).hex() == "00800000"


@pytest.mark.parametrize("C,H,W,scale", [(192, 12, 20, 1.5), (128, 3, 5, 0.3), (8, 1, 1, 3.0), (320, 17, 30, 6.0)])
def test_rans_channel_rows_bit_exact(lic, C, H, W, scale):
    L = 32
    cdf = O.cdf_table(RNG.uniform(0.5, 1.5, C), L)
    sym = np.clip(np.round(RNG.standard_normal((C, H, W)) * scale), -L, L).astype(np.int8)
    ref = O.rans_encode(sym, O.channel_rows(sym.shape), cdf)
    got = lic.rans_encode(sym, cdf)
    assert got == ref
    assert np.array_equal(lic.rans_decode(got, sym.shape, cdf), sym)
    assert np.array_equal(O.rans_decode(got, O.channel_rows(sym.shape), cdf).reshape(sym.shape), sym)


def test_rans_indexed_rows_bit_exact(lic):
    L = 32
    cdf = O.cdf_table(scale_table(), L)
    n = 200_000
    idx = RNG.integers(0, 64, n).astype(np.uint8)
    sig = scale_table()[idx]
    sym = np.clip(np.round(RNG.standard_normal(n) * sig * 0.7), -L, L).astype(np.int8)
    ref = O.rans_encode(sym, idx.astype(np.int32), cdf)
    got = lic.rans_encode(sym, cdf, rows=idx)
    assert got == ref
    assert np.array_equal(lic.rans_decode(got, (n,), cdf, rows=idx), sym)


def test_rans_corrupt(lic):
    L = 32
    cdf = O.cdf_table([1.0, 2.0, 4.0], L)
    sym = np.clip(np.round(RNG.standard_normal((3, 16, 16)) * 2), -L, L).astype(np.int8)
    b = lic.rans_encode(sym, cdf)
    for cut in (1, 3, len(b) // 2):
        with pytest.raises(lic.CorruptStream):
            lic.rans_decode(b[:-cut], sym.shape, cdf)
    with pytest.raises(lic.CorruptStream):
        lic.rans_decode(b + b"\x01", sym.shape, cdf)
    with pytest.raises(lic.LicError):
        lic.rans_encode(np.full((3, 1, 1), 40, np.int8), cdf)      # outside [-L, L]


def test_licw_roundtrip():
    for kind in (0, 1):
        spec = ModelSpec(kind=kind, N=128, M=192)
        w = generate_weights(spec, 5)
        blob = write_licw(spec, w)
        spec2, w2 = read_licw_blocks(blob)
        assert spec2 == spec
        assert all(np.array_equal(w[k], w2[k]) for k in w)
        assert write_licw(spec, generate_weights(spec, 5)) == blob          # deterministic
        assert blob[:4] == b"LICW"


@pytest.mark.parametrize("C,H,W,scale", [(192, 12, 20, 1.5), (128, 3, 5, 0.3), (320, 17, 30, 6.0)])
def test_fast_coder_channel_rows_bit_exact(lic, C, H, W, scale):
    """Prepared tables (reciprocal encode, bucketed decode) emit the oracle's bytes."""
    L = 32
    cdf = O.cdf_table(RNG.uniform(0.5, 1.5, C), L)
    sym = np.clip(np.round(RNG.standard_normal((C, H, W)) * scale), -L, L).astype(np.int8)
    t = lic.RansTables(cdf)
    b = t.encode(sym)
    assert b == O.rans_encode(sym, O.channel_rows(sym.shape), cdf)
    assert np.array_equal(t.decode(b, sym.shape), sym)


def test_fast_coder_indexed_rows_bit_exact(lic):
    L = 32
    cdf = O.cdf_table(scale_table(), L)
    n = 300_000
    idx = RNG.integers(0, 64, n).astype(np.uint8)
    sym = np.clip(np.round(RNG.standard_normal(n) * scale_table()[idx]), -L, L).astype(np.int8)
    sym[:1000] = 32                      # freq-1 edge symbols (reciprocal special case)
    sym[1000:2000] = -32
    t = lic.RansTables(cdf)
    b = t.encode(sym, rows=idx)
    assert b == O.rans_encode(sym, idx.astype(np.int32), cdf)
    assert np.array_equal(t.decode(b, (n,), rows=idx), sym)
    with pytest.raises(lic.CorruptStream):
        t.decode(b[:-2], (n,), rows=idx)


def test_fast_coder_general_tables(lic):
    """Arbitrary tables incl. freq-1 and large-freq symbols (known answers)."""
    c = np.array([[0, 100, 40000, 65536]], np.uint32)
    t = lic.RansTables(c, sym_min=0)
    assert t.encode(np.array([2, 1, 0, 1, 2, 2, 1, 1], np.int8), rows=np.zeros(8, np.uint8)).hex() == "009dc5b89250"
    c = np.array([[0, 1, 65536]], np.uint32)
    t = lic.RansTables(c, sym_min=0)
    assert t.encode(np.array([0], np.int8), rows=np.zeros(1, np.uint8)).hex() == "008000000000"
    sym = RNG.integers(0, 2, 5000).astype(np.int8)
    b = t.encode(sym, rows=np.zeros(5000, np.uint8))
    assert b == O.rans_encode(sym, np.zeros(5000), c, sym_min=0)


# ---------------------------------------------------------------- channel-slab substreams (R21)
@pytest.mark.parametrize("C,H,W,K", [(192, 48, 80, 4), (192, 12, 20, 8), (128, 3, 5, 3), (10, 7, 9, 4),
                                     (5, 4, 4, 5), (192, 2, 3, 1), (64, 1, 1, 64),
                                     (192, 48, 80, 16), (320, 12, 20, 32), (192, 3, 7, 16), (48, 8, 8, 16),
                                     (192, 48, 80, 64), (192, 12, 20, 32), (320, 6, 10, 64), (128, 5, 4, 48)])
def test_slab_substreams_channel_rows_bit_exact(lic, C, H, W, K):
    """Product lic_rans_encode_slabs == oracle rans_encode_slabs byte for byte (ragged slabs
    when K does not divide C), lossless through both decoders."""
    L = 32
    cdf = O.cdf_table(RNG.uniform(0.5, 1.5, C), L)
    sym = np.clip(np.round(RNG.standard_normal((C, H, W)) * 1.3), -L, L).astype(np.int8)
    t = lic.RansTables(cdf)
    b = t.encode(sym, substreams=K)
    assert b == O.rans_encode_slabs(sym, None, cdf, K)
    assert np.array_equal(t.decode(b, sym.shape, substreams=K), sym)
    assert np.array_equal(O.rans_decode_slabs(b, sym.shape, None, cdf, K), sym)


@pytest.mark.parametrize("K", [1, 2, 4, 6, 8, 16, 32, 64])
def test_slab_substreams_indexed_rows_bit_exact(lic, K):
    """K a multiple of 16 with equal slabs runs the AVX-512 coder where the CPU has it (same bytes)."""
    L = 32
    cdf = O.cdf_table(scale_table(), L)
    C, H, W = 192, 24, 40
    idx = RNG.integers(0, 64, (C, H, W)).astype(np.uint8)
    sym = np.clip(np.round(RNG.standard_normal((C, H, W)) * scale_table()[idx] * 0.5), -L, L).astype(np.int8)
    sym[0, 0, :] = 32                     # freq-1 edge symbols in the first and last slab
    sym[-1, -1, :] = -32
    t = lic.RansTables(cdf)
    b = t.encode(sym, rows=idx, substreams=K)
    assert b == O.rans_encode_slabs(sym, idx, cdf, K)
    assert np.array_equal(t.decode(b, sym.shape, rows=idx, substreams=K), sym)


def test_slab_substreams_corrupt(lic):
    L = 32
    C = 16
    cdf = O.cdf_table(RNG.uniform(0.5, 1.5, C), L)
    sym = np.clip(np.round(RNG.standard_normal((C, 8, 8)) * 2), -L, L).astype(np.int8)
    t = lic.RansTables(cdf)
    b = t.encode(sym, substreams=4)
    for bad in (b[:-1], b + b"\x00", b[:10]):
        with pytest.raises(lic.CorruptStream):
            t.decode(bad, sym.shape, substreams=4)
    # a length field pointing past the end
    bb = bytearray(b)
    bb[0:4] = (len(b)).to_bytes(4, "big")
    with pytest.raises(lic.CorruptStream):
        t.decode(bytes(bb), sym.shape, substreams=4)
    with pytest.raises(lic.LicError):
        t.encode(sym, substreams=C + 1)   # more slabs than channels


@pytest.mark.parametrize("K", [16, 32, 64])
def test_slab_substreams_simd_corrupt_fuzz(lic, K):
    """Damaged K = 16..64 strings (the vectorised decoder's lanes) fail cleanly: truncation and
    trailing bytes are corrupt; flipped bytes either fail or decode to some symbols, never read
    outside the string."""
    L = 32
    rng = np.random.default_rng(99)
    cdf = O.cdf_table(scale_table(), L)
    C, H, W = 192, 6, 10
    idx = rng.integers(0, 64, (C, H, W)).astype(np.uint8)
    sym = np.clip(np.round(rng.standard_normal((C, H, W)) * scale_table()[idx] * 0.5), -L, L).astype(np.int8)
    t = lic.RansTables(cdf)
    b = t.encode(sym, rows=idx, substreams=K)
    assert np.array_equal(t.decode(b, sym.shape, rows=idx, substreams=K), sym)
    for bad in (b[:-1], b + b"\x00", b[:4 * K + 6]):
        with pytest.raises(lic.CorruptStream):
            t.decode(bad, sym.shape, rows=idx, substreams=K)
    for _ in range(200):
        bb = bytearray(b)
        for pos in rng.integers(4 * K, len(bb), 3):
            bb[pos] ^= int(rng.integers(1, 256))
        try:
            t.decode(bytes(bb), sym.shape, rows=idx, substreams=K)
        except lic.CorruptStream:
            pass


@pytest.mark.parametrize("K", [1, 2, 16])
def test_zero_frequency_symbol_rejected(lic, K):
    """A table may hold zero-frequency entries (lic_rans_prepare accepts them), but a symbol
    with frequency 0 cannot be coded: every encoder (plain, slabs, AVX-512 lanes) returns
    LIC_EINVAL, like lic_rans_encode, instead of a stream that does not decode."""
    L = 2
    row = np.array([0, 100, 100, 65000, 65436, 65536], np.uint32)          # symbol -1 has frequency 0
    cdf = np.stack([row] * 16)
    t = lic.RansTables(cdf, sym_min=-L)
    sym = np.zeros((16, 4, 4), np.int8)
    sym[3, 1, 2] = -1
    with pytest.raises(lic.LicError) as e:
        t.encode(sym, substreams=K)
    assert e.value.status == lic.LIC_EINVAL
    with pytest.raises(lic.LicError):
        lic.rans_encode(sym, cdf, sym_min=-L)
    sym[3, 1, 2] = 1                                                        # nonzero frequency: fine
    data = t.encode(sym, substreams=K)
    assert np.array_equal(t.decode(data, sym.shape, substreams=K), sym)


@pytest.mark.parametrize("K,parts", [(32, 2), (32, 4), (16, 2), (7, 3)])
def test_slab_ranges_compose_the_slab_stream(lic, K, parts):
    """lic_rans_encode_slab_range over a partition of the K slabs, concatenated in order behind
    the K big-endian lengths, is exactly lic_rans_encode_slabs' stream; lic_rans_decode_slab_range
    of every part restores the plane (the pipeline codes one frame's slabs on several threads)."""
    from lic_synth import scale_table
    rng = np.random.default_rng(K * 10 + parts)
    C, H, W = 64, 12, 20
    cdf = lic.cdf_build(scale_table(), 32)
    idx = rng.integers(0, 30, (C, H, W)).astype(np.uint8)
    sym = np.clip(np.round(rng.standard_normal((C, H, W)) * scale_table()[idx]), -32, 32).astype(np.int8)
    t = lic.RansTables(cdf)
    ref = t.encode(sym, idx, substreams=K)
    bounds = [round(p * K / parts) for p in range(parts + 1)]
    strings, lens = [], []
    for kb, ke in zip(bounds[:-1], bounds[1:]):
        s, l = t.encode_range(sym, K, kb, ke, rows=idx)
        strings.append(s)
        lens.extend(int(x) for x in l)
    framed = b"".join(n.to_bytes(4, "big") for n in lens) + b"".join(strings)
    assert framed == ref
    out = np.zeros_like(sym)
    for kb, ke in zip(bounds[:-1], bounds[1:]):
        t.decode_range(ref, sym.shape, K, kb, ke, rows=idx, out=out)
    assert np.array_equal(out, sym)
    with pytest.raises(lic.LicError):
        t.encode_range(sym, K, 3, 3, rows=idx)
