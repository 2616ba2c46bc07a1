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
#include <cstdlib>
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
    bool any_zero = false;          // some (row, symbol) has frequency 0 (cannot be encoded)
};

extern "C" lic_status lic_rans_prepare(const uint32_t* cdf, uint32_t n_rows, uint32_t row_len, int sym_min,
                                       lic_rans_tables** out) {
    if (!cdf || !out || n_rows == 0 || row_len < 2 || row_len > 257) return LIC_EINVAL;
    auto* t = new lic_rans_tables();
    t->n_rows = n_rows; t->row_len = row_len; t->nsym = row_len - 1; t->sym_min = sym_min;
    t->cdf.assign(cdf, cdf + (size_t)n_rows * row_len);
    t->enc.resize((size_t)n_rows * t->nsym);
    t->bucket.resize((size_t)n_rows * 4096 + 4);     // +4: 4-byte gathers of the last entry (AVX-512 path)
    for (uint32_t r = 0; r < n_rows; ++r) {
        const uint32_t* c = &t->cdf[(size_t)r * row_len];
        if (c[0] != 0 || c[t->nsym] != kProbScale) { delete t; return LIC_EINVAL; }
        for (uint32_t s = 0; s < t->nsym; ++s) {
            if (c[s + 1] < c[s]) { delete t; return LIC_EINVAL; }
            const uint32_t start = c[s], freq = c[s + 1] - c[s];
            if (freq == 0) t->any_zero = true;
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

// ------------------------------------------------------------------ channel-slab substreams
// NEXT-2 ("the entropy coding process is highly CPU-intensive",
// :195 faster coders as future work; reading R21).  A C x H x W plane is cut into K
// channel slabs [floor(kC/K), floor((k+1)C/K)); every slab is coded as an independent rANS string
// in exactly the format above.  K = 1 is the plain string; K > 1 frames the strings as K big-endian
// u32 lengths followed by the K strings.  One thread codes the K strings in lockstep (symbol i of
// slab 0, of slab 1, ...): the per-string dependency chains (mulhi / table lookup / renormalise)
// are independent, so they overlap in the core's pipelines instead of running back to back.
namespace {

struct SlabGeom {
    uint32_t K;
    size_t hw;
    size_t begin[64], count[64];       // symbol range of slab k
    uint32_t ch0[64];                   // first channel of slab k
};

bool slab_geom(lic_shape plane, uint32_t K, SlabGeom& g) {
    if (K == 0 || K > 64 || K > (plane.c ? plane.c : 1)) return false;
    g.K = K;
    g.hw = (size_t)plane.h * plane.w;
    for (uint32_t k = 0; k < K; ++k) {
        const uint32_t c0 = (uint32_t)((uint64_t)k * plane.c / K), c1 = (uint32_t)((uint64_t)(k + 1) * plane.c / K);
        g.ch0[k] = c0;
        g.begin[k] = (size_t)c0 * g.hw;
        g.count[k] = (size_t)(c1 - c0) * g.hw;
    }
    return true;
}

#define LIC_INLINE inline __attribute__((always_inline))

// One encoder step (symbol idx) of one string.  kRow: row[idx] per symbol, else the channel,
// tracked by a countdown (ch, rem) instead of a division.  Renormalisation emits at most two
// bytes (x < 2^31, xmax >= 2^15) and is branch-free: the byte is always stored one below the
// pointer, which only advances when it is emitted.
// Table fields are passed by value (locals): the byte stores through uint8_t* may alias any
// memory, so fields read through `t` would be reloaded after every store.
struct EncCtx { const EncSym* enc; uint32_t nsym, nrows; int smin; };
struct DecCtx { const uint32_t* cdf; const uint8_t* bucket; uint32_t row_len, nrows; int smin; };

template <bool kRow>
LIC_INLINE void enc_step(const EncCtx t, const int8_t* sym, const uint8_t* row, size_t hw, size_t idx,
                         uint32_t& x, uint8_t*& ptr, uint32_t& ch, size_t& rem) {
    uint32_t r;
    if (kRow) {
        r = row[idx];
    } else {
        r = ch;
        if (--rem == 0) { --ch; rem = hw; }
    }
    const int s = (int)sym[idx] - t.smin;       // validated by the caller (validate_planes)
    const EncSym e = t.enc[(size_t)r * t.nsym + s];
    uint32_t xv = x;
    uint8_t* pj = ptr;
    pj[-1] = (uint8_t)xv;
    const uint32_t e1 = xv >= e.xmax;
    pj -= e1; xv >>= 8 * e1;
    pj[-1] = (uint8_t)xv;
    const uint32_t e2 = xv >= e.xmax;
    pj -= e2; xv >>= 8 * e2;
    const uint32_t q = (uint32_t)(((uint64_t)xv * e.rcp) >> 32) >> e.shift;
    x = xv + e.bias + q * (uint32_t)e.cmpl;
    ptr = pj;
}

// Encoder: G strings, last symbol to first.  String j writes backwards from hi[j] into a scratch
// region of 2 * count + 8 bytes (<= 2 bytes per symbol + the 4-byte state, so it cannot
// overflow).  Strings longer than the shortest first code their extra tail symbols alone, then
// all G run in lockstep over the common prefix.
template <int G, bool kRow>
lic_status enc_group(const lic_rans_tables* tab, const int8_t* __restrict sym, const uint8_t* __restrict row,
                     const SlabGeom& g, int k0, uint8_t* const* hi, uint8_t** ptr_out) {
    const EncCtx t{tab->enc.data(), tab->nsym, tab->n_rows, tab->sym_min};
    const size_t hw = g.hw ? g.hw : 1;
    uint32_t x[G], ch[G];
    uint8_t* ptr[G];
    size_t rem[G], beg[G];
    size_t nmin = ~size_t(0);
    for (int j = 0; j < G; ++j) {
        const size_t c = g.count[k0 + j];
        x[j] = kRansLow; ptr[j] = hi[j]; beg[j] = g.begin[k0 + j];
        ch[j] = g.ch0[k0 + j] + (uint32_t)(c ? (c - 1) / hw : 0);
        rem[j] = c ? (c - 1) % hw + 1 : 0;
        nmin = std::min(nmin, c);
    }
    for (int j = 0; j < G; ++j)
        for (size_t i = g.count[k0 + j]; i-- > nmin;) enc_step<kRow>(t, sym, row, hw, beg[j] + i, x[j], ptr[j], ch[j], rem[j]);
    for (size_t i = nmin; i-- > 0;) {
#pragma GCC unroll 8
        for (int j = 0; j < G; ++j) enc_step<kRow>(t, sym, row, hw, beg[j] + i, x[j], ptr[j], ch[j], rem[j]);
    }
    for (int j = 0; j < G; ++j) {
        uint8_t* pj = ptr[j];
        *--pj = (uint8_t)x[j];
        *--pj = (uint8_t)(x[j] >> 8);
        *--pj = (uint8_t)(x[j] >> 16);
        *--pj = (uint8_t)(x[j] >> 24);
        ptr_out[j] = pj;
    }
    return LIC_OK;
}

// One decoder step (symbol idx) of one string.  Branch-free renormalisation (at most two bytes:
// x >= 2^7 after the coding step) while two input bytes remain, checked bytes near the end.
// Returns false on a corrupt stream (exhausted input).
template <bool kRow>
LIC_INLINE int dec_step(const DecCtx t, const uint8_t* row, size_t hw, size_t idx, uint32_t& x,
                        const uint8_t*& p, const uint8_t* end, uint32_t& ch, size_t& rem, int8_t* sym_out) {
    uint32_t r;
    if (kRow) {
        r = row[idx];
    } else {
        r = ch;
        if (--rem == 0) { ++ch; rem = hw; }
    }
    const uint32_t* c = t.cdf + (size_t)r * t.row_len;     // r validated by the caller
    uint32_t xv = x;
    const uint32_t slot = xv & (kProbScale - 1);
    uint32_t s = t.bucket[(size_t)r * 4096 + (slot >> 4)];
    while (c[s + 1] <= slot) ++s;
    const uint32_t start = c[s], freq = c[s + 1] - start;
    xv = freq * (xv >> kProbBits) + slot - start;
    const uint8_t* pj = p;
    if (end - pj >= 2) {
        const uint32_t d1 = xv < kRansLow;
        xv = d1 ? (xv << 8) | pj[0] : xv;
        pj += d1;
        const uint32_t d2 = xv < kRansLow;
        xv = d2 ? (xv << 8) | pj[0] : xv;
        pj += d2;
    } else {
        while (xv < kRansLow) {
            if (pj >= end) return LIC_ECORRUPT;
            xv = (xv << 8) | *pj++;
        }
    }
    x = xv;
    p = pj;
    sym_out[idx] = (int8_t)((int)s + t.smin);
    return LIC_OK;
}

// Decoder: G strings in lockstep over the common prefix, then each string's tail alone.
template <int G, bool kRow>
lic_status dec_group(const lic_rans_tables* tab, const uint8_t* const* in, const size_t* len,
                     const uint8_t* __restrict row, const SlabGeom& g, int k0, int8_t* __restrict sym_out) {
    const DecCtx t{tab->cdf.data(), tab->bucket.data(), tab->row_len, tab->n_rows, tab->sym_min};
    const size_t hw = g.hw ? g.hw : 1;
    uint32_t x[G], ch[G];
    const uint8_t* p[G];
    const uint8_t* end[G];
    size_t rem[G], beg[G];
    size_t nmin = ~size_t(0);
    for (int j = 0; j < G; ++j) {
        if (len[j] < 4) return LIC_ECORRUPT;
        const uint8_t* q = in[j];
        x[j] = ((uint32_t)q[0] << 24) | ((uint32_t)q[1] << 16) | ((uint32_t)q[2] << 8) | q[3];
        p[j] = q + 4;
        end[j] = q + len[j];
        ch[j] = g.ch0[k0 + j]; rem[j] = hw; beg[j] = g.begin[k0 + j];
        nmin = std::min(nmin, g.count[k0 + j]);
    }
    for (size_t i = 0; i < nmin; ++i) {
        int st = 0;
#pragma GCC unroll 8
        for (int j = 0; j < G; ++j) st |= dec_step<kRow>(t, row, hw, beg[j] + i, x[j], p[j], end[j], ch[j], rem[j], sym_out);
        if (st) return LIC_ECORRUPT;
    }
    for (int j = 0; j < G; ++j)
        for (size_t i = nmin; i < g.count[k0 + j]; ++i) {
            const int st = dec_step<kRow>(t, row, hw, beg[j] + i, x[j], p[j], end[j], ch[j], rem[j], sym_out);
            if (st) return (lic_status)st;
        }
    for (int j = 0; j < G; ++j)
        if (x[j] != kRansLow || p[j] != end[j]) return LIC_ECORRUPT;
    return LIC_OK;
}

// Range checks hoisted out of the coding loops (vectorisable): every row < n_rows and, for the
// encoder, every symbol inside the table's support.
// rows in range, symbols inside the table, and (tables with zero-frequency entries only)
// every symbol of nonzero frequency in its row: row[i], or the channel i / hw of the plane
bool validate_planes(const lic_rans_tables* t, const int8_t* sym, const uint8_t* row, size_t n, size_t hw) {
    uint32_t bad = 0;
    if (row) {
        const uint8_t nr = (uint8_t)std::min<uint32_t>(t->n_rows, 255);
        const uint32_t big = t->n_rows > 255;
        for (size_t i = 0; i < n; ++i) bad |= (uint32_t)(row[i] >= nr) & (big ^ 1u);
    }
    if (sym) {
        const int smin = t->sym_min, ns = (int)t->nsym;
        for (size_t i = 0; i < n; ++i) bad |= (uint32_t)((unsigned)((int)sym[i] - smin) >= (unsigned)ns);
        if (bad == 0 && t->any_zero) {
            for (size_t i = 0; i < n && !bad; ++i) {
                const size_t r = row ? row[i] : (hw ? i / hw : 0);
                if (r >= t->n_rows || t->enc[r * t->nsym + (size_t)((int)sym[i] - smin)].xmax == 0) bad = 1;
            }
        }
    }
    return bad == 0;
}

// ------------------------------------------------------------------ AVX-512: 16 strings per thread
// The 16 channel-slab strings of a group are coded in the 16 lanes of a vector (state x, input /
// output offsets, table lookups by gather).  Same bitstream as the scalar coder: each lane runs the
// exact scalar recurrence.  Used when the slabs of a group are equal (C % K == 0) and the CPU has
// AVX-512 (env LIC_NO_AVX512=1 disables); the first (encoder) / last (decoder) few symbols of
// every string, where 4-byte gathers could read past an array, run through the scalar steps.
#if defined(__x86_64__) && defined(__GNUC__)
#include <immintrin.h>
#define LIC_AVX512 __attribute__((target("avx512f,avx512bw,avx512vl,avx512dq")))

bool use_avx512() {
    static const bool ok = [] {
        const char* e = std::getenv("LIC_NO_AVX512");
        if (e && e[0] == '1') return false;
        __builtin_cpu_init();
        return __builtin_cpu_supports("avx512f") && __builtin_cpu_supports("avx512bw") &&
               __builtin_cpu_supports("avx512vl") && __builtin_cpu_supports("avx512dq");
    }();
    return ok;
}

bool simd_group_ok(const SlabGeom& g, uint32_t k0, int nl) {
    const size_t n = g.count[k0];
    if (n < 16 || n % 4 || n * (size_t)nl >= (1ull << 31)) return false;
    for (int j = 1; j < nl; ++j)
        if (g.count[k0 + j] != n || g.begin[k0 + j] != g.begin[k0] + (size_t)j * n) return false;
    return true;
}

// V vectors of 16 lanes (16V strings): V independent dependency chains per step hide the
// gather latencies of one chain (slot -> bucket -> cdf -> state -> renormalisation).
template <int V>
LIC_AVX512 lic_status dec_avx512(const lic_rans_tables* tab, const uint8_t* base, const uint8_t* const* in,
                                 const size_t* len, const uint8_t* row, const SlabGeom& g, int k0, int8_t* sym_out) {
    constexpr int NL = 16 * V;
    const size_t n = g.count[k0], hw = g.hw ? g.hw : 1;
    alignas(64) uint32_t xs[NL], off[NL], endo[NL], chs[NL];
    for (int j = 0; j < NL; ++j) {
        if (len[j] < 4) return LIC_ECORRUPT;
        const uint8_t* q = in[j];
        xs[j] = ((uint32_t)q[0] << 24) | ((uint32_t)q[1] << 16) | ((uint32_t)q[2] << 8) | q[3];
        off[j] = (uint32_t)(q + 4 - base);
        endo[j] = (uint32_t)(q + len[j] - base);
        chs[j] = g.ch0[k0 + j];
    }
    const int* cdf = reinterpret_cast<const int*>(tab->cdf.data());
    const void* bucket = tab->bucket.data();
    __m512i x[V], vo[V], ve[V], ch0[V], slab[V];
    const __m512i lanes = _mm512_setr_epi32(0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 15);
    for (int v = 0; v < V; ++v) {
        x[v] = _mm512_load_si512(xs + 16 * v);
        vo[v] = _mm512_load_si512(off + 16 * v);
        ve[v] = _mm512_load_si512(endo + 16 * v);
        ch0[v] = _mm512_load_si512(chs + 16 * v);
        slab[v] = _mm512_mullo_epi32(_mm512_add_epi32(lanes, _mm512_set1_epi32(16 * v)), _mm512_set1_epi32((int)n));
    }
    const __m512i L = _mm512_set1_epi32((int)kRansLow), m16 = _mm512_set1_epi32(0xFFFF), ff = _mm512_set1_epi32(0xFF);
    const __m512i one = _mm512_set1_epi32(1), rl = _mm512_set1_epi32((int)tab->row_len);
    const __m512i smin = _mm512_set1_epi32(tab->sym_min), twelve = _mm512_set1_epi32(12);
    const uint8_t* rowg = row ? row + g.begin[k0] : nullptr;
    int8_t* outg = sym_out + g.begin[k0];
    size_t i = 0;
    // de-interleave two vectors of 8 (lo, hi) dword pairs into 16 lo / 16 hi dwords
    const __m512i even = _mm512_setr_epi32(0, 2, 4, 6, 8, 10, 12, 14, 16, 18, 20, 22, 24, 26, 28, 30);
    const __m512i odd = _mm512_setr_epi32(1, 3, 5, 7, 9, 11, 13, 15, 17, 19, 21, 23, 25, 27, 29, 31);
    for (; i + 8 <= n; i += 4) {
        // <= 8 input bytes per lane in 4 steps, 4-byte gather windows: stop 12 bytes before an end
        __mmask16 low = 0;
        for (int v = 0; v < V; ++v) low |= _mm512_cmplt_epu32_mask(_mm512_sub_epi32(ve[v], vo[v]), twelve);
        if (low) break;
        __m512i w[V], rows4[V];
        for (int v = 0; v < V; ++v) {
            w[v] = _mm512_setzero_si512();
            if (rowg) rows4[v] = _mm512_i32gather_epi32(slab[v], rowg + i, 1);     // rows of steps i .. i+3
        }
        for (int u = 0; u < 4; ++u) {
            const size_t ii = i + u;
            const __m512i chv = _mm512_set1_epi32((int)(ii / hw));
#pragma GCC unroll 4
            for (int v = 0; v < V; ++v) {
                const __m512i r = rowg ? _mm512_and_si512(_mm512_srli_epi32(rows4[v], 8 * u), ff)
                                       : _mm512_add_epi32(ch0[v], chv);
                const __m512i slot = _mm512_and_si512(x[v], m16);
                const __m512i bidx = _mm512_add_epi32(_mm512_slli_epi32(r, 12), _mm512_srli_epi32(slot, 4));
                __m512i s = _mm512_and_si512(_mm512_i32gather_epi32(bidx, bucket, 1), ff);
                const __m512i cb = _mm512_mullo_epi32(r, rl);
                __m512i st, nxt;
                for (;;) {                   // (c[s], c[s + 1]) pairs by 64-bit gathers; c[s + 1] <= slot: next
                    const __m512i ci = _mm512_add_epi32(cb, s);
                    const __m512i p0 = _mm512_i32gather_epi64(_mm512_castsi512_si256(ci), cdf, 4);
                    const __m512i p1 = _mm512_i32gather_epi64(_mm512_extracti64x4_epi64(ci, 1), cdf, 4);
                    st = _mm512_permutex2var_epi32(p0, even, p1);
                    nxt = _mm512_permutex2var_epi32(p0, odd, p1);
                    const __mmask16 m = _mm512_cmple_epu32_mask(nxt, slot);
                    if (!m) break;
                    s = _mm512_mask_add_epi32(s, m, s, one);
                }
                __m512i xv = _mm512_add_epi32(_mm512_mullo_epi32(_mm512_sub_epi32(nxt, st), _mm512_srli_epi32(x[v], 16)),
                                              _mm512_sub_epi32(slot, st));
                // at most two renormalisation bytes, both from one 4-byte gather
                const __mmask16 m1 = _mm512_cmplt_epu32_mask(xv, L);
                const __m512i b4 = _mm512_mask_i32gather_epi32(_mm512_setzero_si512(), m1, vo[v], base, 1);
                xv = _mm512_mask_or_epi32(xv, m1, _mm512_slli_epi32(xv, 8), _mm512_and_si512(b4, ff));
                const __mmask16 m2 = _mm512_cmplt_epu32_mask(xv, L);              // subset of m1
                xv = _mm512_mask_or_epi32(xv, m2, _mm512_slli_epi32(xv, 8), _mm512_and_si512(_mm512_srli_epi32(b4, 8), ff));
                vo[v] = _mm512_mask_add_epi32(vo[v], m1, vo[v], one);
                vo[v] = _mm512_mask_add_epi32(vo[v], m2, vo[v], one);
                x[v] = xv;
                w[v] = _mm512_or_si512(w[v], _mm512_slli_epi32(_mm512_and_si512(_mm512_add_epi32(s, smin), ff), 8 * u));
            }
        }
        for (int v = 0; v < V; ++v) _mm512_i32scatter_epi32(outg + i, slab[v], w[v], 1);
    }
    // scalar continuation of every lane
    for (int v = 0; v < V; ++v) {
        _mm512_store_si512(xs + 16 * v, x[v]);
        _mm512_store_si512(off + 16 * v, vo[v]);
    }
    const DecCtx t{tab->cdf.data(), tab->bucket.data(), tab->row_len, tab->n_rows, tab->sym_min};
    for (int j = 0; j < NL; ++j) {
        uint32_t xv = xs[j], ch = g.ch0[k0 + j] + (uint32_t)(i / hw);
        size_t rem = hw - i % hw;
        const uint8_t* pj = base + off[j];
        const uint8_t* end = base + endo[j];
        const size_t b0 = g.begin[k0 + j];
        for (size_t ii = i; ii < n; ++ii) {
            const int st = row ? dec_step<true>(t, row, hw, b0 + ii, xv, pj, end, ch, rem, sym_out)
                               : dec_step<false>(t, row, hw, b0 + ii, xv, pj, end, ch, rem, sym_out);
            if (st) return (lic_status)st;
        }
        if (xv != kRansLow || pj != end) return LIC_ECORRUPT;
    }
    return LIC_OK;
}

template <int V>
LIC_AVX512 lic_status enc_avx512(const lic_rans_tables* tab, const int8_t* sym, const uint8_t* row,
                                 const SlabGeom& g, int k0, uint8_t* base, uint8_t* const* hi, uint8_t** ptr_out) {
    constexpr int NL = 16 * V;
    const size_t n = g.count[k0], hw = g.hw ? g.hw : 1;
    const EncCtx t{tab->enc.data(), tab->nsym, tab->n_rows, tab->sym_min};
    alignas(64) uint32_t xs[NL], off[NL], chs[NL];
    // scalar head: the last 4 symbols of every string (4-byte gathers stay inside the planes below)
    const size_t head = 4;
    for (int j = 0; j < NL; ++j) {
        uint32_t xv = kRansLow, ch = g.ch0[k0 + j] + (uint32_t)((n - 1) / hw);
        size_t rem = (n - 1) % hw + 1;
        uint8_t* pj = hi[j];
        for (size_t ii = n; ii-- > n - head;)
            row ? enc_step<true>(t, sym, row, hw, g.begin[k0 + j] + ii, xv, pj, ch, rem)
                : enc_step<false>(t, sym, row, hw, g.begin[k0 + j] + ii, xv, pj, ch, rem);
        xs[j] = xv;
        off[j] = (uint32_t)(pj - base);
        chs[j] = g.ch0[k0 + j];
    }
    const int* enc = reinterpret_cast<const int*>(tab->enc.data());
    __m512i x[V], vp[V], ch0[V], slab[V];
    const __m512i lanes = _mm512_setr_epi32(0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 15);
    for (int v = 0; v < V; ++v) {
        x[v] = _mm512_load_si512(xs + 16 * v);
        vp[v] = _mm512_load_si512(off + 16 * v);
        ch0[v] = _mm512_load_si512(chs + 16 * v);
        slab[v] = _mm512_mullo_epi32(_mm512_add_epi32(lanes, _mm512_set1_epi32(16 * v)), _mm512_set1_epi32((int)n));
    }
    const __m512i ff = _mm512_set1_epi32(0xFF), one = _mm512_set1_epi32(1), two = _mm512_set1_epi32(2);
    const __m512i three = _mm512_set1_epi32(3);
    const __m512i nsym = _mm512_set1_epi32((int)tab->nsym), smin = _mm512_set1_epi32(tab->sym_min);
    const __m512i m16 = _mm512_set1_epi32(0xFFFF);
    const uint8_t* rowg = row ? row + g.begin[k0] : nullptr;
    const int8_t* symg = sym + g.begin[k0];
    const __m512i even = _mm512_setr_epi32(0, 2, 4, 6, 8, 10, 12, 14, 16, 18, 20, 22, 24, 26, 28, 30);
    const __m512i odd = _mm512_setr_epi32(1, 3, 5, 7, 9, 11, 13, 15, 17, 19, 21, 23, 25, 27, 29, 31);
    // groups of 4 symbols (n - head is a multiple of 4): rows and symbols of steps i0 .. i0+3 from one
    // 4-byte gather each, coded i0+3 first
    for (size_t i0 = n - head; i0 >= 4;) {
        i0 -= 4;
        __m512i rows4[V], syms4[V];
        for (int v = 0; v < V; ++v) {
            if (rowg) rows4[v] = _mm512_i32gather_epi32(slab[v], rowg + i0, 1);
            syms4[v] = _mm512_i32gather_epi32(slab[v], symg + i0, 1);
        }
        for (int u = 3; u >= 0; --u) {
            const size_t i = i0 + (size_t)u;
            const __m512i chv = _mm512_set1_epi32((int)(i / hw));
#pragma GCC unroll 4
            for (int v = 0; v < V; ++v) {
                const __m512i r = rowg ? _mm512_and_si512(_mm512_srli_epi32(rows4[v], 8 * u), ff)
                                       : _mm512_add_epi32(ch0[v], chv);
                const __m512i sv = _mm512_srai_epi32(_mm512_slli_epi32(syms4[v], 24 - 8 * u), 24);
                const __m512i e4 = _mm512_slli_epi32(_mm512_add_epi32(_mm512_mullo_epi32(r, nsym), _mm512_sub_epi32(sv, smin)), 2);
                // EncSym = {xmax, rcp} {bias, cmpl | shift << 16}: two 64-bit gathers per half
                const __m512i e2 = _mm512_add_epi32(e4, two);
                const __m512i a0 = _mm512_i32gather_epi64(_mm512_castsi512_si256(e4), enc, 4);
                const __m512i a1 = _mm512_i32gather_epi64(_mm512_extracti64x4_epi64(e4, 1), enc, 4);
                const __m512i b0 = _mm512_i32gather_epi64(_mm512_castsi512_si256(e2), enc, 4);
                const __m512i b1 = _mm512_i32gather_epi64(_mm512_extracti64x4_epi64(e2, 1), enc, 4);
                const __m512i xmax = _mm512_permutex2var_epi32(a0, even, a1);
                const __m512i rcp = _mm512_permutex2var_epi32(a0, odd, a1);
                const __m512i bias = _mm512_permutex2var_epi32(b0, even, b1);
                const __m512i cs = _mm512_permutex2var_epi32(b0, odd, b1);
                __m512i xv = x[v];
                for (int rn = 0; rn < 2; ++rn) {             // at most two renormalisation bytes, emitted downwards
                    const __mmask16 m = _mm512_cmpge_epu32_mask(xv, xmax);
                    vp[v] = _mm512_mask_sub_epi32(vp[v], m, vp[v], one);
                    // a 4-byte store whose top byte lands at the new pointer (the 3 bytes below belong
                    // to this lane's region and are rewritten later or lie outside the string)
                    _mm512_mask_i32scatter_epi32(base, m, _mm512_sub_epi32(vp[v], three), _mm512_slli_epi32(xv, 24), 1);
                    xv = _mm512_mask_srli_epi32(xv, m, xv, 8);
                }
                const __m512i pe = _mm512_srli_epi64(_mm512_mul_epu32(xv, rcp), 32);
                const __m512i po = _mm512_mul_epu32(_mm512_srli_epi64(xv, 32), _mm512_srli_epi64(rcp, 32));
                const __m512i q = _mm512_srlv_epi32(_mm512_mask_blend_epi32(0xAAAA, pe, po), _mm512_srli_epi32(cs, 16));
                x[v] = _mm512_add_epi32(_mm512_add_epi32(xv, bias), _mm512_mullo_epi32(q, _mm512_and_si512(cs, m16)));
            }
        }
    }
    for (int v = 0; v < V; ++v) {
        _mm512_store_si512(xs + 16 * v, x[v]);
        _mm512_store_si512(off + 16 * v, vp[v]);
    }
    for (int j = 0; j < NL; ++j) {
        uint8_t* pj = base + off[j];
        *--pj = (uint8_t)xs[j];
        *--pj = (uint8_t)(xs[j] >> 8);
        *--pj = (uint8_t)(xs[j] >> 16);
        *--pj = (uint8_t)(xs[j] >> 24);
        ptr_out[j] = pj;
    }
    return LIC_OK;
}

// largest vector group (V = 4, 2, 1 x 16 strings) that fits the remaining slabs
int simd_lanes(const SlabGeom& g, uint32_t k0, uint32_t left) {
    if (!use_avx512()) return 0;
    for (int nl = 64; nl >= 16; nl >>= 1)
        if ((int)left >= nl && simd_group_ok(g, k0, nl)) return nl;
    return 0;
}
#else
int simd_lanes(const SlabGeom&, uint32_t, uint32_t) { return 0; }
#endif

inline void put_be32(uint8_t* q, uint32_t v) {
    q[0] = (uint8_t)(v >> 24); q[1] = (uint8_t)(v >> 16); q[2] = (uint8_t)(v >> 8); q[3] = (uint8_t)v;
}
inline uint32_t get_be32(const uint8_t* q) {
    return ((uint32_t)q[0] << 24) | ((uint32_t)q[1] << 16) | ((uint32_t)q[2] << 8) | q[3];
}

}  // namespace

namespace {

// Slabs [kb, ke) of a K-slab plane: the strings (in the per-thread scratch, start[k]..hi[k])
lic_status encode_slab_range(const lic_rans_tables* t, const int8_t* sym, const uint8_t* row, const SlabGeom& g,
                             uint32_t kb, uint32_t ke, std::vector<uint8_t>& scratch, uint8_t** start, uint8_t** hi) {
    // per-slab scratch regions: 2 bytes per symbol + 8 (renormalisation emits <= 16 bits per symbol)
    size_t need = 0;
    size_t off[64];
    for (uint32_t k = kb; k < ke; ++k) { off[k] = need; need += 2 * g.count[k] + 8; }
    if (scratch.size() < need) scratch.resize(need);
    for (uint32_t k = kb; k < ke; ++k) hi[k] = scratch.data() + off[k] + 2 * g.count[k] + 8;
    for (uint32_t k0 = kb; k0 < ke;) {
        const uint32_t left = ke - k0;
#if defined(__x86_64__) && defined(__GNUC__)
        if (const int nl = simd_lanes(g, k0, left)) {
            const lic_status st = nl == 64 ? enc_avx512<4>(t, sym, row, g, (int)k0, scratch.data(), hi + k0, start + k0)
                                : nl == 32 ? enc_avx512<2>(t, sym, row, g, (int)k0, scratch.data(), hi + k0, start + k0)
                                           : enc_avx512<1>(t, sym, row, g, (int)k0, scratch.data(), hi + k0, start + k0);
            if (st) return st;
            k0 += (uint32_t)nl;
            continue;
        }
#endif
        const int G = left >= 4 ? 4 : left >= 2 ? 2 : 1;
        lic_status st;
        if (row) {
            st = G == 4 ? enc_group<4, true>(t, sym, row, g, (int)k0, hi + k0, start + k0)
               : G == 2 ? enc_group<2, true>(t, sym, row, g, (int)k0, hi + k0, start + k0)
                        : enc_group<1, true>(t, sym, row, g, (int)k0, hi + k0, start + k0);
        } else {
            st = G == 4 ? enc_group<4, false>(t, sym, row, g, (int)k0, hi + k0, start + k0)
               : G == 2 ? enc_group<2, false>(t, sym, row, g, (int)k0, hi + k0, start + k0)
                        : enc_group<1, false>(t, sym, row, g, (int)k0, hi + k0, start + k0);
        }
        if (st) return st;
        k0 += (uint32_t)G;
    }
    return LIC_OK;
}

lic_status decode_slab_range(const lic_rans_tables* t, const uint8_t* in, const uint8_t* const* sp, const size_t* sl,
                             const uint8_t* row, const SlabGeom& g, uint32_t kb, uint32_t ke, int8_t* sym_out) {
    for (uint32_t k0 = kb; k0 < ke;) {
        const uint32_t left = ke - k0;
#if defined(__x86_64__) && defined(__GNUC__)
        if (const int nl = simd_lanes(g, k0, left)) {
            const lic_status st = nl == 64 ? dec_avx512<4>(t, in, sp + k0, sl + k0, row, g, (int)k0, sym_out)
                                : nl == 32 ? dec_avx512<2>(t, in, sp + k0, sl + k0, row, g, (int)k0, sym_out)
                                           : dec_avx512<1>(t, in, sp + k0, sl + k0, row, g, (int)k0, sym_out);
            if (st) return st;
            k0 += (uint32_t)nl;
            continue;
        }
#endif
        const int G = left >= 4 ? 4 : left >= 2 ? 2 : 1;
        lic_status st;
        if (row) {
            st = G == 4 ? dec_group<4, true>(t, sp + k0, sl + k0, row, g, (int)k0, sym_out)
               : G == 2 ? dec_group<2, true>(t, sp + k0, sl + k0, row, g, (int)k0, sym_out)
                        : dec_group<1, true>(t, sp + k0, sl + k0, row, g, (int)k0, sym_out);
        } else {
            st = G == 4 ? dec_group<4, false>(t, sp + k0, sl + k0, row, g, (int)k0, sym_out)
               : G == 2 ? dec_group<2, false>(t, sp + k0, sl + k0, row, g, (int)k0, sym_out)
                        : dec_group<1, false>(t, sp + k0, sl + k0, row, g, (int)k0, sym_out);
        }
        if (st) return st;
        k0 += (uint32_t)G;
    }
    return LIC_OK;
}

// the K big-endian lengths of a framed slab string -> string pointers / lengths
lic_status parse_slab_frame(const uint8_t* in, size_t len, uint32_t K, const uint8_t** sp, size_t* sl) {
    if (!in || len < 4 * (size_t)K) return LIC_ECORRUPT;
    size_t pos = 4 * (size_t)K;
    for (uint32_t k = 0; k < K; ++k) {
        sl[k] = get_be32(in + 4 * k);
        if (sl[k] > len - pos) return LIC_ECORRUPT;
        sp[k] = in + pos;
        pos += sl[k];
    }
    return pos == len ? LIC_OK : LIC_ECORRUPT;
}

}  // namespace

extern "C" lic_status lic_rans_encode_slabs(const lic_rans_tables* t, const int8_t* sym, const uint8_t* row,
                                            lic_shape plane, uint32_t K, uint8_t* out, size_t cap, size_t* out_len) {
    if (!t || !out || !out_len) return LIC_EINVAL;
    if (K <= 1) return lic_rans_encode_fast(t, sym, row, plane, out, cap, out_len);
    SlabGeom g;
    if (!slab_geom(plane, K, g)) return LIC_EINVAL;
    if (g.hw * plane.c && !sym) return LIC_EINVAL;
    if (!validate_planes(t, sym, row, g.hw * plane.c, g.hw)) return LIC_EINVAL;
    if (!row && plane.c > t->n_rows) return LIC_EINVAL;
    thread_local std::vector<uint8_t> scratch;
    uint8_t* hi[64]; uint8_t* start[64];
    if (lic_status st = encode_slab_range(t, sym, row, g, 0, K, scratch, start, hi)) return st;
    size_t total = 4 * (size_t)K;
    for (uint32_t k = 0; k < K; ++k) total += (size_t)(hi[k] - start[k]);
    if (total > cap) return LIC_ENOSPACE;
    uint8_t* w = out + 4 * (size_t)K;
    for (uint32_t k = 0; k < K; ++k) {
        const size_t n = (size_t)(hi[k] - start[k]);
        put_be32(out + 4 * k, (uint32_t)n);
        std::memcpy(w, start[k], n);
        w += n;
    }
    *out_len = total;
    return LIC_OK;
}

extern "C" lic_status lic_rans_encode_slab_range(const lic_rans_tables* t, const int8_t* sym, const uint8_t* row,
                                                 lic_shape plane, uint32_t K, uint32_t k_begin, uint32_t k_end,
                                                 uint8_t* out, size_t cap, uint32_t* lens, size_t* out_len) {
    if (!t || !out || !out_len || !lens || K < 1 || k_begin >= k_end || k_end > K) return LIC_EINVAL;
    SlabGeom g;
    if (!slab_geom(plane, K, g)) return LIC_EINVAL;
    if (g.hw * plane.c && !sym) return LIC_EINVAL;
    // the range's channels only (row[] and sym[] are whole-plane arrays)
    const size_t b0 = g.begin[k_begin], n = g.begin[k_end - 1] + g.count[k_end - 1] - b0;
    if (!validate_planes(t, sym + b0, row ? row + b0 : nullptr, n, g.hw)) return LIC_EINVAL;
    if (!row && (uint32_t)((uint64_t)k_end * plane.c / K) > t->n_rows) return LIC_EINVAL;
    thread_local std::vector<uint8_t> scratch;
    uint8_t* hi[64]; uint8_t* start[64];
    if (lic_status st = encode_slab_range(t, sym, row, g, k_begin, k_end, scratch, start, hi)) return st;
    size_t total = 0;
    for (uint32_t k = k_begin; k < k_end; ++k) total += (size_t)(hi[k] - start[k]);
    if (total > cap) return LIC_ENOSPACE;
    uint8_t* w = out;
    for (uint32_t k = k_begin; k < k_end; ++k) {
        const size_t m = (size_t)(hi[k] - start[k]);
        lens[k - k_begin] = (uint32_t)m;
        std::memcpy(w, start[k], m);
        w += m;
    }
    *out_len = total;
    return LIC_OK;
}

extern "C" lic_status lic_rans_decode_slabs(const lic_rans_tables* t, const uint8_t* in, size_t len, const uint8_t* row,
                                            lic_shape plane, uint32_t K, int8_t* sym_out) {
    if (!t) return LIC_EINVAL;
    if (K <= 1) return lic_rans_decode_fast(t, in, len, row, plane, sym_out);
    return lic_rans_decode_slab_range(t, in, len, row, plane, K, 0, K, sym_out);
}

extern "C" lic_status lic_rans_decode_slab_range(const lic_rans_tables* t, const uint8_t* in, size_t len,
                                                 const uint8_t* row, lic_shape plane, uint32_t K, uint32_t k_begin,
                                                 uint32_t k_end, int8_t* sym_out) {
    if (!t || K < 2 || k_begin >= k_end || k_end > K) return LIC_EINVAL;
    SlabGeom g;
    if (!slab_geom(plane, K, g)) return LIC_EINVAL;
    if (g.hw * plane.c && !sym_out) return LIC_EINVAL;
    const size_t b0 = g.begin[k_begin], n = g.begin[k_end - 1] + g.count[k_end - 1] - b0;
    if (!validate_planes(t, nullptr, row ? row + b0 : nullptr, n, g.hw)) return LIC_EINVAL;
    if (!row && (uint32_t)((uint64_t)k_end * plane.c / K) > t->n_rows) return LIC_EINVAL;
    const uint8_t* sp[64];
    size_t sl[64];
    if (lic_status st = parse_slab_frame(in, len, K, sp, sl)) return st;
    return decode_slab_range(t, in, sp, sl, row, g, k_begin, k_end, sym_out);
}
