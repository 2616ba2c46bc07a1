// host_coder.cpp -- the host half of the codec: CDF tables and the rANS coder.
//
// The paper keeps entropy coding on the CPU ("The entropy coding process is highly
// CPU-intensive"; it integrates CompressAI's rANS coder) and
// overlaps it with the GPU transforms via the pipeline.  This file is the
// product coder (reentrant, no globals); the oracle has its own independent copy.
//
// CDF rows (reading R8): zero-mean discretised Gaussian
// over k in [-L, L] with the tails folded into +-L, quantised to 16 bits with every
// frequency >= 1 and the rounding residue given to k = 0.  Evaluated in fp64 exactly as
// written: tail(t) = erfc((t) / sqrt(2)) / 2 with t = (|k| -+ 1/2) / sigma.
//
// rANS: 32-bit state, lower bound 2^23, byte renormalisation,
// 16-bit precision; symbols encoded last-to-first so the decoder runs first-to-last;
// the final state is flushed as 4 big-endian bytes at the front.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <vector>

#include "../../include/lic.h"

namespace {

constexpr uint32_t kProbBits = 16;
constexpr uint32_t kProbScale = 1u << kProbBits;
constexpr uint32_t kRansLow = 1u << 23;

// upper-tail mass P(X > t*sigma) of a unit Gaussian at t, i.e. Phi(-t)
inline double upper_tail(double t) { return 0.5 * std::erfc(t / std::sqrt(2.0)); }

bool build_row(double sigma, int L, uint32_t* cdf) {
    if (!(sigma > 0.0) || L < 1) return false;
    const int n = 2 * L + 1;
    std::vector<int64_t> freq(n);
    int64_t total = 0;
    for (int k = -L; k <= L; ++k) {
        const int a = k < 0 ? -k : k;
        double p;
        if (a == 0)
            p = 1.0 - 2.0 * upper_tail(0.5 / sigma);
        else if (a < L)
            p = upper_tail((a - 0.5) / sigma) - upper_tail((a + 0.5) / sigma);
        else
            p = upper_tail((a - 0.5) / sigma);            // folded tail
        int64_t f = (int64_t)std::nearbyint(p * (double)kProbScale);  // ties to even
        if (f < 1) f = 1;
        freq[k + L] = f;
        total += f;
    }
    freq[L] += (int64_t)kProbScale - total;
    if (freq[L] < 1) return false;
    uint32_t acc = 0;
    cdf[0] = 0;
    for (int i = 0; i < n; ++i) {
        acc += (uint32_t)freq[i];
        cdf[i + 1] = acc;
    }
    return acc == kProbScale;
}

inline uint32_t row_of(const uint8_t* row, size_t i, size_t plane_hw) {
    return row ? (uint32_t)row[i] : (uint32_t)(i / plane_hw);
}

}  // namespace

extern "C" lic_status lic_cdf_build(const float* sigmas, uint32_t n, uint32_t L, uint32_t* out) {
    if (!sigmas || !out || L < 1 || L > 127) return LIC_EINVAL;
    const uint32_t len = 2 * L + 2;
    for (uint32_t i = 0; i < n; ++i)
        if (!build_row((double)sigmas[i], (int)L, out + (size_t)i * len)) return LIC_EINVAL;
    return LIC_OK;
}

extern "C" lic_status lic_rans_encode(const int8_t* sym, const uint8_t* row, lic_shape plane,
                                      const uint32_t* cdf, uint32_t n_rows, uint32_t row_len,
                                      int sym_min, uint8_t* out, size_t cap, size_t* out_len) {
    if (!cdf || !out || !out_len || row_len < 2 || n_rows == 0) return LIC_EINVAL;
    const size_t hw = (size_t)plane.h * plane.w;
    const size_t n = hw * plane.c;
    if (n && !sym) return LIC_EINVAL;
    const int nsym = (int)row_len - 1;
    // bytes are produced back to front; write them at the tail of `out` and move once
    size_t pos = cap;
    uint32_t x = kRansLow;
    for (size_t i = n; i-- > 0;) {
        const uint32_t r = row_of(row, i, hw ? hw : 1);
        const int s = (int)sym[i] - sym_min;
        if (r >= n_rows || s < 0 || s >= nsym) return LIC_EINVAL;
        const uint32_t* c = cdf + (size_t)r * row_len;
        const uint32_t start = c[s];
        const uint32_t freq = c[s + 1] - start;
        if (freq == 0) return LIC_EINVAL;
        // renormalise so the coding step below keeps x < 2^31
        const uint32_t bound = ((kRansLow >> kProbBits) << 8) * freq;
        while (x >= bound) {
            if (pos == 0) return LIC_ENOSPACE;
            out[--pos] = (uint8_t)x;
            x >>= 8;
        }
        const uint32_t q = x / freq;
        x = (q << kProbBits) + (x - q * freq) + start;
    }
    if (pos < 4) return LIC_ENOSPACE;
    out[--pos] = (uint8_t)x;
    out[--pos] = (uint8_t)(x >> 8);
    out[--pos] = (uint8_t)(x >> 16);
    out[--pos] = (uint8_t)(x >> 24);
    const size_t len = cap - pos;
    if (pos) std::memmove(out, out + pos, len);
    *out_len = len;
    return LIC_OK;
}

extern "C" lic_status lic_rans_decode(const uint8_t* in, size_t len, const uint8_t* row,
                                      lic_shape plane, const uint32_t* cdf, uint32_t n_rows,
                                      uint32_t row_len, int sym_min, int8_t* sym_out) {
    if (!cdf || row_len < 2 || n_rows == 0) return LIC_EINVAL;
    if (!in || len < 4) return LIC_ECORRUPT;
    const size_t hw = (size_t)plane.h * plane.w;
    const size_t n = hw * plane.c;
    if (n && !sym_out) return LIC_EINVAL;
    uint32_t x = ((uint32_t)in[0] << 24) | ((uint32_t)in[1] << 16) | ((uint32_t)in[2] << 8) | in[3];
    size_t pos = 4;
    const int nsym = (int)row_len - 1;
    for (size_t i = 0; i < n; ++i) {
        const uint32_t r = row_of(row, i, hw ? hw : 1);
        if (r >= n_rows) return LIC_EINVAL;
        const uint32_t* c = cdf + (size_t)r * row_len;
        const uint32_t slot = x & (kProbScale - 1);
        // largest s with c[s] <= slot (c[0] = 0, c[nsym] = 2^16 > slot)
        const uint32_t* hit = std::upper_bound(c, c + nsym + 1, slot);
        const int s = (int)(hit - c) - 1;
        if (s < 0 || s >= nsym) return LIC_ECORRUPT;
        const uint32_t start = c[s], freq = c[s + 1] - c[s];
        if (freq == 0) return LIC_ECORRUPT;
        x = freq * (x >> kProbBits) + slot - start;
        while (x < kRansLow) {
            if (pos >= len) return LIC_ECORRUPT;
            x = (x << 8) | in[pos++];
        }
        sym_out[i] = (int8_t)(s + sym_min);
    }
    if (x != kRansLow || pos != len) return LIC_ECORRUPT;
    return LIC_OK;
}

// ------------------------------------------------------------------ prepared tables
// Encoder: x' = (x / f << 16) + x % f + start = x + start + q * (2^16 - f) with q = x / f
// computed exactly as mulhi(x, rcp) >> shift (x < 2^31 after renormalisation); f = 1 uses
// rcp = 2^32 - 1, shift 0, bias start + 2^16 - 1, which gives q = x - 1 and the same x'.
struct EncSym {
    uint32_t xmax;       // renormalise while x >= xmax
    uint32_t rcp;        // reciprocal of freq
    uint32_t bias;       // start (or start + 2^16 - 1 for freq == 1)
    uint16_t cmpl;       // 2^16 - freq
    uint16_t shift;      // reciprocal shift
};

struct lic_rans_tables {
    uint32_t n_rows = 0, row_len = 0, nsym = 0;
    int sym_min = 0;
    std::vector<uint32_t> cdf;
    std::vector<EncSym> enc;        // n_rows x nsym
    std::vector<uint8_t> bucket;    // n_rows x 4096: symbol holding slot (u << 4)
};

extern "C" lic_status lic_rans_prepare(const uint32_t* cdf, uint32_t n_rows, uint32_t row_len, int sym_min,
                                       lic_rans_tables** out) {
    if (!cdf || !out || n_rows == 0 || row_len < 2 || row_len > 257) return LIC_EINVAL;
    auto* t = new lic_rans_tables();
    t->n_rows = n_rows; t->row_len = row_len; t->nsym = row_len - 1; t->sym_min = sym_min;
    t->cdf.assign(cdf, cdf + (size_t)n_rows * row_len);
    t->enc.resize((size_t)n_rows * t->nsym);
    t->bucket.resize((size_t)n_rows * 4096);
    for (uint32_t r = 0; r < n_rows; ++r) {
        const uint32_t* c = &t->cdf[(size_t)r * row_len];
        if (c[0] != 0 || c[t->nsym] != kProbScale) { delete t; return LIC_EINVAL; }
        for (uint32_t s = 0; s < t->nsym; ++s) {
            if (c[s + 1] < c[s]) { delete t; return LIC_EINVAL; }
            const uint32_t start = c[s], freq = c[s + 1] - c[s];
            EncSym& e = t->enc[(size_t)r * t->nsym + s];
            e.xmax = ((kRansLow >> kProbBits) << 8) * freq;
            e.cmpl = (uint16_t)((kProbScale - freq) & 0xFFFF);
            if (freq < 2) {
                e.rcp = ~0u; e.shift = 0; e.bias = start + kProbScale - 1;
            } else {
                uint32_t sh = 0;
                while (freq > (1u << sh)) ++sh;
                e.rcp = (uint32_t)(((1ull << (sh + 31)) + freq - 1) / freq);
                e.shift = (uint16_t)(sh - 1);
                e.bias = start;
            }
        }
        uint32_t s = 0;
        for (uint32_t u = 0; u < 4096; ++u) {
            const uint32_t slot = u << 4;
            while (c[s + 1] <= slot) ++s;
            t->bucket[(size_t)r * 4096 + u] = (uint8_t)s;
        }
    }
    *out = t;
    return LIC_OK;
}

extern "C" void lic_rans_tables_free(lic_rans_tables* t) { delete t; }

extern "C" lic_status lic_rans_encode_fast(const lic_rans_tables* t, const int8_t* sym, const uint8_t* row,
                                           lic_shape plane, uint8_t* out, size_t cap, size_t* out_len) {
    if (!t || !out || !out_len) return LIC_EINVAL;
    const size_t hw = (size_t)plane.h * plane.w;
    const size_t n = hw * plane.c;
    if (n && !sym) return LIC_EINVAL;
    const EncSym* enc = t->enc.data();
    const uint32_t nsym = t->nsym, nrows = t->n_rows;
    const int smin = t->sym_min;
    uint8_t* ptr = out + cap;
    uint32_t x = kRansLow;
    size_t i = n;
    // channel-row planes: iterate channel by channel so the row lookup is hoisted
    while (i > 0) {
        const size_t seg_end = i;
        const size_t seg_begin = row ? 0 : ((i - 1) / (hw ? hw : 1)) * (hw ? hw : 1);
        const uint32_t crow = row ? 0 : (uint32_t)((i - 1) / (hw ? hw : 1));
        if (!row && crow >= nrows) return LIC_EINVAL;
        for (size_t j = seg_end; j-- > seg_begin;) {
            const uint32_t r = row ? row[j] : crow;
            const int s = (int)sym[j] - smin;
            if (r >= nrows || (unsigned)s >= nsym) return LIC_EINVAL;
            const EncSym& e = enc[(size_t)r * nsym + s];
            if (e.xmax == 0) return LIC_EINVAL;
            while (x >= e.xmax) {
                if (ptr == out) return LIC_ENOSPACE;
                *--ptr = (uint8_t)x;
                x >>= 8;
            }
            const uint32_t q = (uint32_t)(((uint64_t)x * e.rcp) >> 32) >> e.shift;
            x = x + e.bias + q * (uint32_t)e.cmpl;
        }
        i = seg_begin;
    }
    if ((size_t)(ptr - out) < 4) return LIC_ENOSPACE;
    *--ptr = (uint8_t)x;
    *--ptr = (uint8_t)(x >> 8);
    *--ptr = (uint8_t)(x >> 16);
    *--ptr = (uint8_t)(x >> 24);
    const size_t len = (size_t)(out + cap - ptr);
    if (ptr != out) std::memmove(out, ptr, len);
    *out_len = len;
    return LIC_OK;
}

extern "C" lic_status lic_rans_decode_fast(const lic_rans_tables* t, const uint8_t* in, size_t len,
                                           const uint8_t* row, lic_shape plane, int8_t* sym_out) {
    if (!t) return LIC_EINVAL;
    if (!in || len < 4) return LIC_ECORRUPT;
    const size_t hw = (size_t)plane.h * plane.w;
    const size_t n = hw * plane.c;
    if (n && !sym_out) return LIC_EINVAL;
    const uint32_t* cdf = t->cdf.data();
    const uint8_t* bucket = t->bucket.data();
    const uint32_t rl = t->row_len, nrows = t->n_rows;
    const int smin = t->sym_min;
    uint32_t x = ((uint32_t)in[0] << 24) | ((uint32_t)in[1] << 16) | ((uint32_t)in[2] << 8) | in[3];
    const uint8_t* p = in + 4;
    const uint8_t* end = in + len;
    for (size_t i = 0; i < n; ++i) {
        const uint32_t r = row ? row[i] : (uint32_t)(i / hw);
        if (r >= nrows) return LIC_EINVAL;
        const uint32_t* c = cdf + (size_t)r * rl;
        const uint32_t slot = x & (kProbScale - 1);
        uint32_t s = bucket[(size_t)r * 4096 + (slot >> 4)];
        while (c[s + 1] <= slot) ++s;        // c[nsym] = 2^16 > slot terminates the scan
        const uint32_t start = c[s], freq = c[s + 1] - start;
        x = freq * (x >> kProbBits) + slot - start;
        while (x < kRansLow) {
            if (p >= end) return LIC_ECORRUPT;
            x = (x << 8) | *p++;
        }
        sym_out[i] = (int8_t)((int)s + smin);
    }
    if (x != kRansLow || p != end) return LIC_ECORRUPT;
    return LIC_OK;
}
