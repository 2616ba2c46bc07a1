"""CPU oracle of the rans64 coder with bypass escape.

TEST INFRASTRUCTURE ONLY: may be imported only by ``tests/``, ``__graft_entry__.smoke()``
and ``bench.py``'s reference legs.  It never imports the product package and the product
never imports it.  Plain Python integers, one symbol at a time, in the order the coder is
defined (R23); meant for inputs of a few thousand symbols.

What it follows: the paper's implementations B and C "simply integrate the CompressAI entropy
coder [8] into our system", i.e. ryg_rans' 64-bit rANS plus CompressAI's
escape ("bypass") coding of values outside a table's support.  DESIGN.md R23 writes that scheme out; this file is that
reading, step by step:

* state x: 64-bit, L = 2^31, renormalisation in 32-bit words, precision 16;
* a table row r is a quantised CDF c_r[0 .. n_r-1] (c_r[0] = 0, c_r[n_r-1] = 2^16); values
  v = s - offset_r in [0, n_r-2) are ordinary symbols, v_max = n_r - 2 is the escape;
* an escaped value carries raw = -2v-1 (v < 0) or 2(v - v_max) (v >= v_max), sent as
  n_bypass 4-bit chunks (n_bypass = number of 4-bit digits of raw, itself sent as 4-bit
  chunks where 15 means "15 more follow"), each chunk put with probability 2^-4;
* symbols are pushed in order and coded in reverse (rANS is LIFO); the final state is
  flushed as two little-endian u32 words (low, high) in front of the renormalisation words.

Parity status: pinned by tests/test_rans64.py -- states worked out by hand from the
definitions (no renormalisation, one escape), the CDF quantiser on hand examples, the
ideal code length bound, and round trips.
"""
from __future__ import annotations

import struct

import numpy as np

PRECISION = 16
RANS64_L = 1 << 31
BYPASS_PRECISION = 4
MAX_BYPASS_VAL = (1 << BYPASS_PRECISION) - 1
_M64 = (1 << 64) - 1


class CorruptStream(Exception):
    pass


def pmf_to_quantized_cdf(pmf, precision=PRECISION):
    """Quantised CDF of `pmf` (the last entry is the escape's tail mass), R23 (c):
    round each p * 2^precision (float32, half away from zero), rescale so the sum is 2^precision, prefix-sum, pin the last
    entry to 2^precision, then give every zero-frequency symbol one slot taken from the
    smallest frequency > 1 (shifting the CDF entries between the two)."""
    one = 1 << precision
    # float32 product, rounded half away from zero (p >= 0)
    f = [int(np.floor(float(np.float32(p) * np.float32(one)) + 0.5)) for p in pmf]
    cdf = [0] + f
    total = sum(cdf)
    if total == 0:
        raise ValueError("pmf sums to zero")
    cdf = [(one * c) // total for c in cdf]
    for i in range(1, len(cdf)):
        cdf[i] += cdf[i - 1]
    cdf[-1] = one
    n = len(cdf)
    for i in range(n - 1):
        if cdf[i] == cdf[i + 1]:
            best_freq, best = None, -1
            for j in range(n - 1):
                fj = cdf[j + 1] - cdf[j]
                if fj > 1 and (best_freq is None or fj < best_freq):
                    best_freq, best = fj, j
            if best < 0:
                raise ValueError("no frequency to steal")
            if best < i:
                for j in range(best + 1, i + 1):
                    cdf[j] -= 1
            else:
                for j in range(i + 1, best + 1):
                    cdf[j] += 1
    return np.array(cdf, np.uint32)


def _enc_put(x, out, start, freq):
    x_max = ((RANS64_L >> PRECISION) << 32) * freq
    if x >= x_max:
        out.append(x & 0xFFFFFFFF)
        x >>= 32
    return ((x // freq) << PRECISION) + (x % freq) + start


def _enc_put_bits(x, out, val, nbits):
    freq = 1 << (PRECISION - nbits)
    x_max = ((RANS64_L >> PRECISION) << 32) * freq
    if x >= x_max:
        out.append(x & 0xFFFFFFFF)
        x >>= 32
    return (x << nbits) | val


def symbol_list(sym, idx, cdfs, sizes, offsets):
    """The pushed symbols in order: (start, freq, bypass)."""
    syms = []
    for s, r in zip(sym, idx):
        s, r = int(s), int(r)
        cdf = cdfs[r]
        vmax = int(sizes[r]) - 2
        v = s - int(offsets[r])
        raw = 0
        if v < 0:
            raw, v = -2 * v - 1, vmax
        elif v >= vmax:
            raw, v = 2 * (v - vmax), vmax
        syms.append((int(cdf[v]), int(cdf[v + 1]) - int(cdf[v]), False))
        if v == vmax:
            nb = 0
            while raw >> (nb * BYPASS_PRECISION):
                nb += 1
            val = nb
            while val >= MAX_BYPASS_VAL:
                syms.append((MAX_BYPASS_VAL, 1, True))
                val -= MAX_BYPASS_VAL
            syms.append((val, 1, True))
            for j in range(nb):
                syms.append(((raw >> (j * BYPASS_PRECISION)) & MAX_BYPASS_VAL, 1, True))
    return syms


def rans64_encode(sym, idx, cdfs, sizes, offsets) -> bytes:
    """Encode symbols `sym` (ints) with table rows `idx`; returns the byte string."""
    x = RANS64_L
    words = []                          # renormalisation words in emission order
    for start, freq, bypass in reversed(symbol_list(sym, idx, cdfs, sizes, offsets)):
        if bypass:
            x = _enc_put_bits(x, words, start, BYPASS_PRECISION)
        else:
            x = _enc_put(x, words, start, freq)
        assert 0 <= x <= _M64
    # flush: the stream is read front to back, so the last emitted word comes first
    return struct.pack("<II", x & 0xFFFFFFFF, x >> 32) + b"".join(struct.pack("<I", w) for w in reversed(words))


def rans64_decode(data: bytes, idx, cdfs, sizes, offsets):
    """Inverse of rans64_encode; CorruptStream when the words run out, a slot falls outside
    a table, or the final state is not L with every word consumed."""
    if len(data) % 4 or len(data) < 8:
        raise CorruptStream("length")
    w = list(struct.unpack(f"<{len(data) // 4}I", data))
    x = w[0] | (w[1] << 32)
    pos = 2

    def refill(x):
        nonlocal pos
        if x < RANS64_L:
            if pos >= len(w):
                raise CorruptStream("exhausted")
            x = (x << 32) | w[pos]
            pos += 1
        return x

    def get_bits(x, n):
        val = x & ((1 << n) - 1)
        return refill(x >> n), val

    out = []
    for r in idx:
        r = int(r)
        cdf = cdfs[r]
        n = int(sizes[r])
        vmax = n - 2
        cum = x & ((1 << PRECISION) - 1)
        s = None
        for k in range(n - 1):
            if int(cdf[k + 1]) > cum:
                s = k
                break
        if s is None:
            raise CorruptStream("slot")
        start, freq = int(cdf[s]), int(cdf[s + 1]) - int(cdf[s])
        x = refill(freq * (x >> PRECISION) + (x & ((1 << PRECISION) - 1)) - start)
        v = s
        if v == vmax:
            x, val = get_bits(x, BYPASS_PRECISION)
            nb = val
            while val == MAX_BYPASS_VAL:
                x, val = get_bits(x, BYPASS_PRECISION)
                nb += val
            if nb > 16:
                raise CorruptStream("escape length")
            raw = 0
            for j in range(nb):
                x, val = get_bits(x, BYPASS_PRECISION)
                raw |= val << (j * BYPASS_PRECISION)
            v = raw >> 1
            v = -v - 1 if raw & 1 else v + vmax
        out.append(v + int(offsets[r]))
    if x != RANS64_L or pos != len(w):
        raise CorruptStream("final state")
    return np.array(out, np.int64)


def ideal_bits(sym, idx, cdfs, sizes, offsets):
    """Information content of the pushed symbols: sum of -log2(freq / 2^16) (bypass chunks:
    4 bits each)."""
    bits = 0.0
    for start, freq, bypass in symbol_list(sym, idx, cdfs, sizes, offsets):
        bits += BYPASS_PRECISION if bypass else PRECISION - np.log2(freq)
    return bits


def gaussian_tables(scales, tail_mass=1e-9, stride=None):
    """CompressAI's GaussianConditional tables (R23 (d)), fp64: m = -Phi^-1(tail_mass / 2);
    row r covers k = -c .. c with c = ceil(scale_r * m); p_k = Phi((1/2 - |k|) / s) -
    Phi((-1/2 - |k|) / s); the escape carries both tails 2 Phi((-1/2 - c) / s); offsets -c."""
    import math
    from statistics import NormalDist

    m = -NormalDist().inv_cdf(tail_mass / 2)

    def phi(x):
        return 0.5 * math.erfc(-x / math.sqrt(2.0))

    rows, sizes, offsets = [], [], []
    for s in np.asarray(scales, np.float32):
        s = float(s)
        c = int(math.ceil(s * m))
        pmf = [np.float32(phi((0.5 - abs(k)) / s) - phi((-0.5 - abs(k)) / s)) for k in range(-c, c + 1)]
        pmf.append(np.float32(2.0 * phi((-0.5 - c) / s)))
        rows.append(pmf_to_quantized_cdf(pmf))
        sizes.append(2 * c + 3)
        offsets.append(-c)
    if stride is None:
        stride = max(sizes)
    cdfs = np.zeros((len(rows), stride), np.uint32)
    for r, row in enumerate(rows):
        cdfs[r, : row.size] = row
    return cdfs, np.array(sizes, np.int32), np.array(offsets, np.int32)
