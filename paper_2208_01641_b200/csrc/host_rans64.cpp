// host_rans64.cpp -- the rans64 coder with bypass escape.
//
// The paper's implementations B and C "simply integrate the CompressAI entropy coder [8]"
// (PAPER.md:129).  That coder is ryg_rans' 64-bit rANS with CompressAI's escape coding of
// values outside a table's support; reading R23 writes the scheme out and this
// file implements it (the oracle, oracle/rans64.py, is an independent plain-Python copy):
//   * state 64-bit, L = 2^31, 32-bit renormalisation words, precision 16;
//   * table row r: quantised CDF c[0 .. n_r-1], c[0] = 0, c[n_r-1] = 2^16, every frequency
//     >= 1; v = s - offset_r in [0, n_r - 2) is a symbol, v_max = n_r - 2 the escape;
//   * an escaped value sends raw = -2v-1 (v < 0) or 2(v - v_max) in 4-bit chunks after its
//     chunk count (itself in 4-bit chunks, 15 = "15 more follow"), each at probability 2^-4;
//   * rANS is LIFO: symbols are encoded last to first; the final state is written as two
//     little-endian u32 (low, high) in front of the renormalisation words.
// Reentrant, no globals; the decoder validates every read (LIC_ECORRUPT, never a crash).
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <vector>

#include "../../include/lic.h"

namespace {

constexpr uint32_t kPrec = 16;
constexpr uint64_t kL = 1ull << 31;
constexpr uint32_t kBypassBits = 4;
constexpr uint32_t kMaxBypass = (1u << kBypassBits) - 1;
constexpr int kMaxChunks = 9;                   // int32 values: raw < 2^34, at most 9 chunks

struct Tables {
    const uint32_t* cdfs;
    uint32_t n;
    uint32_t stride;
    const int32_t* sizes;
    const int32_t* offsets;
};

bool valid_tables(const Tables& t) {
    if (!t.cdfs || !t.sizes || !t.offsets || t.n == 0 || t.stride < 3) return false;
    for (uint32_t r = 0; r < t.n; ++r) {
        const int32_t n = t.sizes[r];
        if (n < 3 || (uint32_t)n > t.stride) return false;
        const uint32_t* c = t.cdfs + (size_t)r * t.stride;
        if (c[0] != 0 || c[n - 1] != (1u << kPrec)) return false;
        for (int32_t k = 0; k + 1 < n; ++k)
            if (c[k + 1] <= c[k]) return false;
    }
    return true;
}

// ryg_rans Rans64EncPut / Rans64EncPutBits; words are written downwards from *pp
inline void enc_put(uint64_t& x, uint32_t*& p, uint32_t start, uint32_t freq) {
    const uint64_t x_max = ((kL >> kPrec) << 32) * freq;
    if (x >= x_max) { *--p = (uint32_t)x; x >>= 32; }
    x = ((x / freq) << kPrec) + (x % freq) + start;
}
inline void enc_put_bits(uint64_t& x, uint32_t*& p, uint32_t val) {
    const uint64_t x_max = ((kL >> kPrec) << 32) << (kPrec - kBypassBits);
    if (x >= x_max) { *--p = (uint32_t)x; x >>= 32; }
    x = (x << kBypassBits) | val;
}

}  // namespace

extern "C" lic_status lic_cdf_quantize(const float* pmf, uint32_t n, uint32_t* cdf) {
    if (!pmf || !cdf || n == 0) return LIC_EINVAL;
    const uint32_t one = 1u << kPrec;
    std::vector<uint64_t> c(n + 1);
    c[0] = 0;
    uint64_t total = 0;
    for (uint32_t i = 0; i < n; ++i) {
        if (!(pmf[i] >= 0.0f) || !std::isfinite(pmf[i])) return LIC_EINVAL;
        c[i + 1] = (uint64_t)std::round(pmf[i] * (float)one);     // float product, half away from 0
        total += c[i + 1];
    }
    if (total == 0) return LIC_EINVAL;
    for (uint32_t i = 0; i <= n; ++i) c[i] = ((uint64_t)one * c[i]) / total;
    for (uint32_t i = 1; i <= n; ++i) c[i] += c[i - 1];
    c[n] = one;
    // every zero-frequency symbol takes one slot from the smallest frequency > 1
    for (uint32_t i = 0; i < n; ++i) {
        if (c[i] != c[i + 1]) continue;
        uint64_t best_f = ~0ull;
        int64_t best = -1;
        for (uint32_t j = 0; j < n; ++j) {
            const uint64_t f = c[j + 1] - c[j];
            if (f > 1 && f < best_f) { best_f = f; best = j; }
        }
        if (best < 0) return LIC_EINVAL;
        if (best < (int64_t)i) {
            for (int64_t j = best + 1; j <= (int64_t)i; ++j) --c[j];
        } else {
            for (int64_t j = (int64_t)i + 1; j <= best; ++j) ++c[j];
        }
    }
    for (uint32_t i = 0; i <= n; ++i) cdf[i] = (uint32_t)c[i];
    return LIC_OK;
}

extern "C" lic_status lic_cdf64_gaussian(const float* scales, uint32_t n, double tail_mass, uint32_t* cdfs,
                                         uint32_t stride, int32_t* sizes, int32_t* offsets) {
    if (!scales || !cdfs || !sizes || !offsets || n == 0 || !(tail_mass > 0.0 && tail_mass < 1.0))
        return LIC_EINVAL;
    // multiplier m: Phi(-m) = tail_mass / 2 (bisection on the upper tail, fp64)
    auto upper_tail = [](double t) { return 0.5 * std::erfc(t / std::sqrt(2.0)); };
    double lo = 0.0, hi = 40.0;
    for (int it = 0; it < 200; ++it) {
        const double mid = 0.5 * (lo + hi);
        if (upper_tail(mid) > tail_mass / 2) lo = mid; else hi = mid;
    }
    const double m = hi;
    std::vector<float> pmf;
    for (uint32_t r = 0; r < n; ++r) {
        const double s = scales[r];
        if (!(s > 0.0)) return LIC_EINVAL;
        const int32_t center = (int32_t)std::ceil(s * m);
        const int32_t len = 2 * center + 1;
        if ((uint32_t)len + 2 > stride) return LIC_ENOSPACE;
        pmf.assign((size_t)len + 1, 0.0f);
        // P(|k - center| rounds to sample) with Phi(x) = erfc(-x / sqrt 2) / 2
        auto Phi = [](double x) { return 0.5 * std::erfc(-x / std::sqrt(2.0)); };
        for (int32_t k = 0; k < len; ++k) {
            const double a = std::abs(k - center);
            pmf[k] = (float)(Phi((0.5 - a) / s) - Phi((-0.5 - a) / s));
        }
        pmf[len] = (float)(2.0 * Phi((-0.5 - center) / s));       // both tails: the escape
        uint32_t* row = cdfs + (size_t)r * stride;
        std::fill(row, row + stride, 0u);
        if (lic_status st = lic_cdf_quantize(pmf.data(), (uint32_t)len + 1, row)) return st;
        sizes[r] = len + 2;
        offsets[r] = -center;
    }
    return LIC_OK;
}

extern "C" lic_status lic_rans64_encode(const int32_t* sym, const int32_t* idx, size_t n, const uint32_t* cdfs,
                                        uint32_t n_cdfs, uint32_t stride, const int32_t* sizes,
                                        const int32_t* offsets, uint8_t* out, size_t cap, size_t* out_len) {
    if ((!sym || !idx) && n) return LIC_EINVAL;
    if (!out || !out_len) return LIC_EINVAL;
    const Tables t{cdfs, n_cdfs, stride, sizes, offsets};
    if (!valid_tables(t)) return LIC_EINVAL;
    for (size_t i = 0; i < n; ++i)
        if (idx[i] < 0 || (uint32_t)idx[i] >= n_cdfs) return LIC_EINVAL;
    // every put emits at most one word per 16 bits of information: symbols <= 16 bits,
    // chunks 4 bits; an escape adds at most 1 + 2 + 9 chunks (|raw| < 2^33)
    size_t bound_bits = 64;
    for (size_t i = 0; i < n; ++i) bound_bits += kPrec + 12 * kBypassBits;
    static thread_local std::vector<uint32_t> buf;           // reused: no allocation per plane
    if (buf.size() < bound_bits / 32 + 4) buf.resize(bound_bits / 32 + 4);
    uint32_t* const end = buf.data() + bound_bits / 32 + 4;
    uint32_t* p = end;
    uint64_t x = kL;
    for (size_t i = n; i-- > 0;) {
        const int32_t r = idx[i];
        const uint32_t* c = cdfs + (size_t)r * stride;
        const int64_t vmax = sizes[r] - 2;
        int64_t v = (int64_t)sym[i] - offsets[r];
        uint64_t raw = 0;
        if (v < 0) { raw = (uint64_t)(-2 * v - 1); v = vmax; }
        else if (v >= vmax) { raw = (uint64_t)(2 * (v - vmax)); v = vmax; }
        if (v == vmax) {
            // this symbol's pushes, in push order: escape, count chunks, value chunks --
            // encoded here in reverse
            uint32_t chunks[1 + 8 + kMaxChunks];
            int nc = 0;
            int nb = 0;
            while (nb < kMaxChunks && (raw >> (nb * kBypassBits))) ++nb;
            uint32_t val = (uint32_t)nb;
            while (val >= kMaxBypass) { chunks[nc++] = kMaxBypass; val -= kMaxBypass; }
            chunks[nc++] = val;
            for (int j = 0; j < nb; ++j) chunks[nc++] = (uint32_t)(raw >> (j * kBypassBits)) & kMaxBypass;
            for (int j = nc - 1; j >= 0; --j) enc_put_bits(x, p, chunks[j]);
        }
        enc_put(x, p, c[v], c[v + 1] - c[v]);
    }
    *--p = (uint32_t)(x >> 32);
    *--p = (uint32_t)x;
    const size_t words = (size_t)(end - p);
    if (words * 4 > cap) return LIC_ENOSPACE;
    for (size_t k = 0; k < words; ++k) {                 // little-endian u32 words
        const uint32_t w = p[k];
        out[4 * k + 0] = (uint8_t)w;
        out[4 * k + 1] = (uint8_t)(w >> 8);
        out[4 * k + 2] = (uint8_t)(w >> 16);
        out[4 * k + 3] = (uint8_t)(w >> 24);
    }
    *out_len = words * 4;
    return LIC_OK;
}

extern "C" lic_status lic_rans64_decode(const uint8_t* in, size_t len, const int32_t* idx, size_t n,
                                        const uint32_t* cdfs, uint32_t n_cdfs, uint32_t stride,
                                        const int32_t* sizes, const int32_t* offsets, int32_t* sym_out) {
    if ((!idx || !sym_out) && n) return LIC_EINVAL;
    const Tables t{cdfs, n_cdfs, stride, sizes, offsets};
    if (!valid_tables(t)) return LIC_EINVAL;
    if (!in || len % 4 || len < 8) return LIC_ECORRUPT;
    const size_t nw = len / 4;
    auto word = [&](size_t k) -> uint32_t {
        return (uint32_t)in[4 * k] | ((uint32_t)in[4 * k + 1] << 8) | ((uint32_t)in[4 * k + 2] << 16) |
               ((uint32_t)in[4 * k + 3] << 24);
    };
    uint64_t x = (uint64_t)word(0) | ((uint64_t)word(1) << 32);
    size_t pos = 2;
    bool bad = false;
    auto refill = [&]() {
        if (x < kL) {
            if (pos >= nw) { bad = true; return; }
            x = (x << 32) | word(pos++);
        }
    };
    auto get_bits = [&]() -> uint32_t {
        const uint32_t v = (uint32_t)(x & kMaxBypass);
        x >>= kBypassBits;
        refill();
        return v;
    };
    constexpr uint64_t mask = (1ull << kPrec) - 1;
    for (size_t i = 0; i < n; ++i) {
        const int32_t r = idx[i];
        if (r < 0 || (uint32_t)r >= n_cdfs) return LIC_EINVAL;
        const uint32_t* c = cdfs + (size_t)r * stride;
        const int32_t sz = sizes[r];
        const uint32_t cum = (uint32_t)(x & mask);
        // s: the last entry <= cum (c[0] = 0 <= cum < 2^16 = c[sz-1])
        const int32_t s = (int32_t)(std::upper_bound(c, c + sz, cum) - c) - 1;
        if (s < 0 || s > sz - 2) return LIC_ECORRUPT;
        const uint32_t start = c[s], freq = c[s + 1] - c[s];
        x = freq * (x >> kPrec) + (x & mask) - start;
        refill();
        if (bad) return LIC_ECORRUPT;
        int64_t v = s;
        const int32_t vmax = sz - 2;
        if (s == vmax) {
            uint32_t val = get_bits();
            uint32_t nb = val;
            while (!bad && val == kMaxBypass && nb <= (uint32_t)kMaxChunks) { val = get_bits(); nb += val; }
            if (bad || nb > (uint32_t)kMaxChunks) return LIC_ECORRUPT;
            uint64_t raw = 0;
            for (uint32_t j = 0; j < nb; ++j) raw |= (uint64_t)get_bits() << (j * kBypassBits);
            if (bad) return LIC_ECORRUPT;
            const int64_t h = (int64_t)(raw >> 1);
            v = (raw & 1) ? -h - 1 : h + vmax;
        }
        const int64_t outv = v + offsets[r];
        if (outv < INT32_MIN || outv > INT32_MAX) return LIC_ECORRUPT;
        sym_out[i] = (int32_t)outv;
    }
    if (x != kL || pos != nw) return LIC_ECORRUPT;
    return LIC_OK;
}
