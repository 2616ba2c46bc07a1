/*
 * lic_oracle.c -- the CPU ORACLE for the learned-image-codec hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  The product path
 * (paper_2208_01641_b200/) never links, imports or calls anything here, and this
 * file shares no code, header, table or constant generator with it.
 *
 * Plain, slow, obviously-correct definitions written from the paper
 * and the readings of SURVEY.md §8(c) (listed in
 * DESIGN.md §3).  Tensors are fp32, channel-major C x H x W.  Every
 * output element is accumulated in fp64 in a fixed loop order and rounded once
 * to fp32 (SURVEY.md §8(c) "fp64 accumulation per output element").  No
 * blocking, fusion or reordering.  OpenMP only splits independent output
 * channels across threads (the per-element arithmetic is unchanged).
 *
 * Pins (tests/test_oracle_*.py): SPEC.md worked examples, torch float64
 * F.conv2d / F.conv_transpose2d, the conv/deconv adjoint identity, the
 * fixed-point GDN inverse, hand-derived rANS known answers, brute force.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define OR_OK 0
#define OR_EINVAL 1
#define OR_ECORRUPT 3
#define OR_ENOSPACE 5

/* ------------------------------------------------------------------------ */
/* conv2d: "standard cross-correlation with stride and zero
 * padding", output dims floor((H + 2p - k)/s) + 1.  Layer shapes of g_a / h_a
 * per SPEC.md:319:
 *   out[co][oy][ox] = b[co] + sum_{ci,ky,kx} W[co][ci][ky][kx] * in[ci][s*oy+ky-p][s*ox+kx-p]
 * (SURVEY.md §8(c) step 2).  Weights are out x in x k x k. */
int or_conv2d(const float* in, int Cin, int H, int W,
              const float* w, const float* b, int Cout, int k, int s, int p,
              float* out)
{
    if (Cin <= 0 || H <= 0 || W <= 0 || Cout <= 0 || k <= 0 || s <= 0 || p < 0) return OR_EINVAL;
    int Ho = (H + 2 * p - k) / s + 1, Wo = (W + 2 * p - k) / s + 1;
    if (Ho <= 0 || Wo <= 0) return OR_EINVAL;
    #pragma omp parallel for schedule(dynamic, 1)
    for (int co = 0; co < Cout; ++co) {
        for (int oy = 0; oy < Ho; ++oy) {
            for (int ox = 0; ox < Wo; ++ox) {
                double acc = (double)b[co];
                for (int ci = 0; ci < Cin; ++ci) {
                    for (int ky = 0; ky < k; ++ky) {
                        int iy = s * oy + ky - p;
                        if (iy < 0 || iy >= H) continue;
                        for (int kx = 0; kx < k; ++kx) {
                            int ix = s * ox + kx - p;
                            if (ix < 0 || ix >= W) continue;
                            acc += (double)w[((size_t)(co * Cin + ci) * k + ky) * k + kx] *
                                   (double)in[((size_t)ci * H + iy) * W + ix];
                        }
                    }
                }
                out[((size_t)co * Ho + oy) * Wo + ox] = (float)acc;
            }
        }
    }
    return OR_OK;
}

/* ------------------------------------------------------------------------ */
/* conv2d_transpose: "transposed convolution (gradient-of-conv
 * layout)"; with output_padding op the output is (H-1)s - 2p + k + op
 * (op = 1 so the 5x5/s2/p2 layers double the size).
 *   out[co][oy][ox] = b[co] + sum over {ci, iy, ix, ky, kx : s*iy - p + ky = oy,
 *                                           s*ix - p + kx = ox} W[co][ci][ky][kx] * in[ci][iy][ix]
 * (W stored out x in x k x k). */
int or_deconv2d(const float* in, int Cin, int H, int W,
                const float* w, const float* b, int Cout, int k, int s, int p, int op,
                float* out)
{
    if (Cin <= 0 || H <= 0 || W <= 0 || Cout <= 0 || k <= 0 || s <= 0 || p < 0 || op < 0) return OR_EINVAL;
    int Ho = (H - 1) * s - 2 * p + k + op, Wo = (W - 1) * s - 2 * p + k + op;
    if (Ho <= 0 || Wo <= 0) return OR_EINVAL;
    #pragma omp parallel for schedule(dynamic, 1)
    for (int co = 0; co < Cout; ++co) {
        for (int oy = 0; oy < Ho; ++oy) {
            for (int ox = 0; ox < Wo; ++ox) {
                double acc = (double)b[co];
                for (int ci = 0; ci < Cin; ++ci) {
                    for (int ky = 0; ky < k; ++ky) {
                        int ty = oy + p - ky;              /* = s*iy */
                        if (ty < 0 || ty % s != 0) continue;
                        int iy = ty / s;
                        if (iy >= H) continue;
                        for (int kx = 0; kx < k; ++kx) {
                            int tx = ox + p - kx;
                            if (tx < 0 || tx % s != 0) continue;
                            int ix = tx / s;
                            if (ix >= W) continue;
                            acc += (double)w[((size_t)(co * Cin + ci) * k + ky) * k + kx] *
                                   (double)in[((size_t)ci * H + iy) * W + ix];
                        }
                    }
                }
                out[((size_t)co * Ho + oy) * Wo + ox] = (float)acc;
            }
        }
    }
    return OR_OK;
}

/* ------------------------------------------------------------------------ */
/* GDN / IGDN: "forward: y_i = x_i / sqrt(beta_i + sum_j gamma_ij x_j^2);
 * inverse: multiply instead of divide" (definition from the paper's [9],
 * PAPER.md:133 "a large portion of the performance overhead lies within the
 * GDN activation function").  n_i accumulated in fp64 over j = 0..C-1. */
int or_gdn(const float* x, int C, int H, int W, const float* beta, const float* gamma,
           int inverse, float* out)
{
    if (C <= 0 || H <= 0 || W <= 0) return OR_EINVAL;
    size_t HW = (size_t)H * W;
    #pragma omp parallel for schedule(dynamic, 1)
    for (int i = 0; i < C; ++i) {
        for (size_t q = 0; q < HW; ++q) {
            double n = (double)beta[i];
            for (int j = 0; j < C; ++j) {
                double xj = (double)x[(size_t)j * HW + q];
                n += (double)gamma[(size_t)i * C + j] * xj * xj;
            }
            double xi = (double)x[(size_t)i * HW + q];
            out[(size_t)i * HW + q] = (float)(inverse ? xi * sqrt(n) : xi / sqrt(n));
        }
    }
    return OR_OK;
}

/* 1DN: "y_i = x_i / (beta_i + sum_j gamma_ij |x_j|); inverse:
 * multiply instead of divide" (the paper's implementation C, PAPER.md:131-137,
 * citing [6]). */
int or_onedn(const float* x, int C, int H, int W, const float* beta, const float* gamma,
             int inverse, float* out)
{
    if (C <= 0 || H <= 0 || W <= 0) return OR_EINVAL;
    size_t HW = (size_t)H * W;
    #pragma omp parallel for schedule(dynamic, 1)
    for (int i = 0; i < C; ++i) {
        for (size_t q = 0; q < HW; ++q) {
            double n = (double)beta[i];
            for (int j = 0; j < C; ++j)
                n += (double)gamma[(size_t)i * C + j] * fabs((double)x[(size_t)j * HW + q]);
            double xi = (double)x[(size_t)i * HW + q];
            out[(size_t)i * HW + q] = (float)(inverse ? xi * n : xi / n);
        }
    }
    return OR_OK;
}

/* ------------------------------------------------------------------------ */
/* Quantise ("quantization of y with a channel-wise mean, producing
 * y-hat"; "symbol s = round(y - mu_c) (ties away from zero, clamped
 * to support); y-hat = s + mu_c").  v = y - mu in fp32; round half
 * away from zero (C roundf); clamp to [-L, L] and count clamped elements (c6).
 * mu == NULL means mu = 0 (hyperprior y). */
int or_quantize(const float* y, int C, int H, int W, const float* mu, int L,
                int8_t* sym, float* yhat, uint64_t* n_sat)
{
    if (C <= 0 || H <= 0 || W <= 0 || L <= 0 || L > 127) return OR_EINVAL;
    size_t HW = (size_t)H * W;
    uint64_t sat = 0;
    for (int c = 0; c < C; ++c) {
        float m = mu ? mu[c] : 0.0f;
        for (size_t q = 0; q < HW; ++q) {
            float v = y[(size_t)c * HW + q] - m;
            float r = roundf(v);
            if (r > (float)L) { r = (float)L; ++sat; }
            if (r < (float)-L) { r = (float)-L; ++sat; }
            if (sym) sym[(size_t)c * HW + q] = (int8_t)r;
            if (yhat) yhat[(size_t)c * HW + q] = r + m;
        }
    }
    if (n_sat) *n_sat = sat;
    return OR_OK;
}

/* Dequantise ("dequantize is exactly symbol + offset"). */
int or_dequantize(const int8_t* sym, int C, int H, int W, const float* mu, float* yhat)
{
    size_t HW = (size_t)H * W;
    for (int c = 0; c < C; ++c) {
        float m = mu ? mu[c] : 0.0f;
        for (size_t q = 0; q < HW; ++q) yhat[(size_t)c * HW + q] = (float)sym[(size_t)c * HW + q] + m;
    }
    return OR_OK;
}

/* ------------------------------------------------------------------------ */
/* scale -> CDF index ("returns the count of table entries
 * strictly less than sigma, clamped to [0, len-1]"; SPEC.md:320 sigma lower
 * bound 0.11).  SURVEY.md c10: sigma' = max(sigma, 0.11f);
 * idx = #{ j in [0, n-2] : table_j < sigma' } (counting only the first n-1
 * entries is the clamp to len-1). */
int or_scale_index(const float* sigma, size_t n, const float* table, int ntab, uint8_t* idx)
{
    if (ntab <= 0 || ntab > 256) return OR_EINVAL;
    for (size_t i = 0; i < n; ++i) {
        float s = sigma[i];
        if (s < 0.11f) s = 0.11f;
        int cnt = 0;
        for (int j = 0; j < ntab - 1; ++j)
            if (table[j] < s) ++cnt;
        idx[i] = (uint8_t)cnt;
    }
    return OR_OK;
}

/* ------------------------------------------------------------------------ */
/* CDF row for a zero-mean discretised Gaussian of scale sigma over k in [-L, L]
 * (readings c7/c8):
 *   p(k)  = Phi(-(|k|-1/2)/sigma) - Phi(-(|k|+1/2)/sigma)      0 < |k| < L
 *   p(0)  = 1 - 2 Phi(-(1/2)/sigma)
 *   p(+-L)= Phi(-(L-1/2)/sigma)                                (tail folded)
 *   Phi(t) = erfc(-t/sqrt(2)) / 2 in fp64
 *   f(k)  = max(1, round_half_even(p(k) * 2^16)); f(0) += 2^16 - sum f
 *   cdf[0] = 0, cdf[i+1] = cdf[i] + f(-L + i)                 (2L+2 entries) */
static double or_phi(double t) { return 0.5 * erfc(-t / sqrt(2.0)); }

int or_cdf_row(double sigma, int L, uint32_t* cdf)
{
    if (!(sigma > 0.0) || L <= 0) return OR_EINVAL;
    int nsym = 2 * L + 1;
    int64_t* f = (int64_t*)malloc(sizeof(int64_t) * (size_t)nsym);
    if (!f) return OR_EINVAL;
    int64_t sum = 0;
    for (int i = 0; i < nsym; ++i) {
        int k = i - L, a = abs(k);
        double p;
        if (a == 0) p = 1.0 - 2.0 * or_phi(-0.5 / sigma);
        else if (a < L) p = or_phi(-(a - 0.5) / sigma) - or_phi(-(a + 0.5) / sigma);
        else p = or_phi(-(a - 0.5) / sigma);
        double q = nearbyint(p * 65536.0);          /* default mode: half to even */
        int64_t fi = (int64_t)q;
        if (fi < 1) fi = 1;
        f[i] = fi;
        sum += fi;
    }
    f[L] += 65536 - sum;
    int ok = f[L] >= 1;
    cdf[0] = 0;
    for (int i = 0; i < nsym; ++i) cdf[i + 1] = cdf[i] + (uint32_t)f[i];
    free(f);
    return ok && cdf[nsym] == 65536u ? OR_OK : OR_EINVAL;
}

/* ------------------------------------------------------------------------ */
/* rANS ("entropy coding"; the coder is CompressAI's rANS,
 * PAPER.md:129; "32-bit-state, byte-renormalizing ... 16-bit CDF
 * precision", SPEC.md:218 big-endian emission):
 *   L_R = 2^23, precision 16.  Encode symbols i = n-1 .. 0 with
 *   (start, freq) = (cdf[row_i][s_i+L], cdf[row_i][s_i+L+1] - start):
 *     while x >= 2^15 * freq: emit(x & 0xFF) to the front, x >>= 8
 *     x = ((x / freq) << 16) + (x % freq) + start
 *   then the 4-byte state, big-endian, at the very front.
 * rows: per-symbol CDF row index; cdf: nrows x row_len; symbol value s sits at
 * CDF index s - sym_min (the codec uses sym_min = -L, row_len = 2L+2; the
 * known-answer tests use sym_min = 0 with arbitrary tables). */
int or_rans_encode(const int8_t* sym, const int32_t* rows, size_t n,
                   const uint32_t* cdf, int nrows, int row_len, int sym_min,
                   uint8_t* out, size_t cap, size_t* out_len)
{
    if (row_len < 2 || nrows <= 0) return OR_EINVAL;
    /* worst case: 2 bytes per symbol + 4 */
    size_t tmpcap = 2 * n + 8;
    uint8_t* tmp = (uint8_t*)malloc(tmpcap);
    if (!tmp) return OR_EINVAL;
    uint8_t* ptr = tmp + tmpcap;
    uint32_t x = 1u << 23;
    for (size_t ii = n; ii-- > 0;) {
        int s = sym[ii] - sym_min, r = rows[ii];
        if (s < 0 || s > row_len - 2 || r < 0 || r >= nrows) { free(tmp); return OR_EINVAL; }
        const uint32_t* c = cdf + (size_t)r * row_len;
        uint32_t start = c[s], freq = c[s + 1] - c[s];
        if (freq == 0) { free(tmp); return OR_EINVAL; }
        uint32_t xmax = (1u << 15) * freq;
        while (x >= xmax) { *--ptr = (uint8_t)(x & 0xFF); x >>= 8; }
        x = ((x / freq) << 16) + (x % freq) + start;
    }
    *--ptr = (uint8_t)(x & 0xFF);
    *--ptr = (uint8_t)((x >> 8) & 0xFF);
    *--ptr = (uint8_t)((x >> 16) & 0xFF);
    *--ptr = (uint8_t)((x >> 24) & 0xFF);
    size_t len = (size_t)(tmp + tmpcap - ptr);
    if (len > cap) { free(tmp); return OR_ENOSPACE; }
    memcpy(out, ptr, len);
    *out_len = len;
    free(tmp);
    return OR_OK;
}

/* Decoder: x = BE32; per symbol slot = x & 0xFFFF,
 * find s with cdf[s] <= slot < cdf[s+1], x = freq*(x>>16) + slot - start,
 * renormalise while x < 2^23 by shifting in the next byte.  At the end require
 * x == 2^23 and every byte consumed; otherwise the stream is corrupt
 * ("explicit corrupt-stream error, never a panic"). */
int or_rans_decode(const uint8_t* in, size_t len, const int32_t* rows, size_t n,
                   const uint32_t* cdf, int nrows, int row_len, int sym_min, int8_t* sym)
{
    if (row_len < 2 || nrows <= 0) return OR_EINVAL;
    if (len < 4) return OR_ECORRUPT;
    size_t pos = 4;
    uint32_t x = ((uint32_t)in[0] << 24) | ((uint32_t)in[1] << 16) | ((uint32_t)in[2] << 8) | in[3];
    for (size_t i = 0; i < n; ++i) {
        int r = rows[i];
        if (r < 0 || r >= nrows) return OR_EINVAL;
        const uint32_t* c = cdf + (size_t)r * row_len;
        uint32_t slot = x & 0xFFFFu;
        int s = -1;
        for (int j = 0; j < row_len - 1; ++j)
            if (c[j] <= slot && slot < c[j + 1]) { s = j; break; }
        if (s < 0) return OR_ECORRUPT;
        uint32_t start = c[s], freq = c[s + 1] - c[s];
        x = freq * (x >> 16) + slot - start;
        while (x < (1u << 23)) {
            if (pos >= len) return OR_ECORRUPT;
            x = (x << 8) | in[pos++];
        }
        sym[i] = (int8_t)(s + sym_min);
    }
    if (x != (1u << 23) || pos != len) return OR_ECORRUPT;
    return OR_OK;
}
