// conv_umma.cu -- the codec's one GEMM engine: persistent, warp-specialised implicit-GEMM
// convolution / transposed convolution on sm_100a tensor cores (tcgen05 + TMEM + TMA)
// with the layer's nonlinearity fused into the epilogue.
//
// What it computes (Fig. 1 transforms; layer list SPEC.md:319):
//   conv   : out[co][oy][ox] = b[co] + sum W[co][ci][ky][kx] in[ci][s*oy+ky-p][s*ox+kx-p]
//   deconv : stride-2 transposed conv (output_padding 1) as 4 sub-pixel phase GEMMs
//            out[co][2qy+py][2qx+px] = b[co] + sum_{taps of phase} W[..][ky][kx] in[ci][qy+dy][qx+dx]
// then one of the EpKind epilogues (GDN per SPEC.md:66 as a second tcgen05 MMA of the
// squared activations against gamma, then rsqrt/sqrt in fp32; quantise per SPEC.md:194;
// sigma -> index per SPEC.md:181-189; clamp per SPEC.md:265).
//
// Data layout: activations NHWC fp16, as two planes hi = fp16(x), lo = fp16(x - hi)
// (DESIGN.md "split-FP16"); weights W[tap][co][ci] fp16 (exact: generator rounds them).
// Each pipeline stage carries one (tap, 64-channel chunk): A_hi, A_lo (128 px x 64 ch,
// loaded by a strided 5-D TMA box so the stride-2 gather and the zero padding are done by
// the TMA unit) and B (BN x 64).  Two MMAs per 16-wide K step (hi, lo) accumulate into the
// same fp32 TMEM accumulator.
//
// Warp roles (256 threads): w0 TMA producer, w1 MMA issuer, w2 TMEM allocator,
// w3 idle, w4-7 epilogue (TMEM lanes 0-127 = the tile's 128 pixels).
#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include "layer.h"
#include "ptx.cuh"

namespace lic {

struct TileCoord { int b, ph, gy0, gx0, nt; };

__device__ __forceinline__ TileCoord decode_tile(const ConvParams& p, int t) {
    TileCoord c;
    c.nt = t % p.n_ntiles;  t /= p.n_ntiles;
    int tx = t % p.tiles_x; t /= p.tiles_x;
    int ty = t % p.tiles_y; t /= p.tiles_y;
    c.ph = t % p.nphase;
    c.b = t / p.nphase;
    c.gx0 = tx * p.Wt;
    c.gy0 = ty * p.Ht;
    return c;
}

// 8 consecutive channels -> one 16-byte fp16 hi vector (+ one lo vector)
__device__ __forceinline__ void split_store8(__half* hi, __half* lo, const float* v) {
    __align__(16) __half h[8];
    __align__(16) __half l[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        h[i] = __float2half_rn(v[i]);
        l[i] = __float2half_rn(v[i] - __half2float(h[i]));
    }
    *reinterpret_cast<uint4*>(hi) = *reinterpret_cast<const uint4*>(h);
    if (lo) *reinterpret_cast<uint4*>(lo) = *reinterpret_cast<const uint4*>(l);
}

// write 32 consecutive channels of one pixel's fp32 values into the swizzled x^2 tile
// (K-major, 128-byte rows, SW128: 16-byte chunk j of row r lives at chunk j ^ (r & 7))
__device__ __forceinline__ void xsq_store32(uint8_t* tile, int row, int col0, const float* v) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        __align__(16) __half h[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) h[i] = __float2half_rn(v[q * 8 + i]);
        int chunk = ((col0 >> 3) + q) ^ (row & 7);
        *reinterpret_cast<uint4*>(tile + row * 128 + chunk * 16) = *reinterpret_cast<const uint4*>(h);
    }
}

__device__ __forceinline__ int round_clamp(float v, int L, int& sat) {
    float r = roundf(v);                 // half away from zero
    if (r > (float)L) { r = (float)L; ++sat; }
    if (r < (float)-L) { r = (float)-L; ++sat; }
    return (int)r;
}

__global__ void __launch_bounds__(256, 1)
conv_umma_kernel(const __grid_constant__ CUtensorMap mapA,
                 const __grid_constant__ CUtensorMap mapB,
                 const __grid_constant__ CUtensorMap mapG,
                 const __grid_constant__ ConvParams p)
{
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + p.off_bar);
    uint64_t* empty_bar = full_bar + p.stages;
    uint64_t* tfull_bar = empty_bar + p.stages;     // [2]
    uint64_t* tempty_bar = tfull_bar + 2;           // [2]
    uint64_t* norm_bar = tempty_bar + 2;
    uint64_t* gamma_bar = norm_bar + 1;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(gamma_bar + 1);

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const bool gdn = (p.ep == EP_GDN || p.ep == EP_IGDN);
    const int nchunk_out = p.BN / 64;               // GDN: BN == Cout, multiple of 64

    if (threadIdx.x == 0) {
        for (int s = 0; s < p.stages; ++s) { mbar_init(&full_bar[s], 1); mbar_init(&empty_bar[s], 1); }
        for (int i = 0; i < 2; ++i) { mbar_init(&tfull_bar[i], 1); mbar_init(&tempty_bar[i], 4); }
        mbar_init(norm_bar, 1);
        mbar_init(gamma_bar, 1);
        fence_mbar_init();
    }
    if (warp == 0 && lane == 0) {
        tma_prefetch_desc(&mapA);
        tma_prefetch_desc(&mapB);
        if (gdn) tma_prefetch_desc(&mapG);
    }
    if (warp == 2) tmem_alloc(tmem_slot, (uint32_t)p.tmem_cols);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    const uint32_t a_bytes = kBM * kBK * 2;          // 16 KB per activation plane
    const uint32_t b_bytes = (uint32_t)p.BN * kBK * 2;
    const uint32_t idesc = idesc_f16_f32(kBM, (uint32_t)p.BN);

    if (warp == 0) {
        // ====================== TMA producer ======================
        if (lane == 0) {
            if (gdn) {
                mbar_arrive_expect_tx(gamma_bar, (uint32_t)nchunk_out * b_bytes);
                for (int c = 0; c < nchunk_out; ++c)
                    tma_load_3d(smem + p.off_gamma + c * b_bytes, &mapG, gamma_bar, c * kBK, 0, 0);
            }
            int stage = 0;
            uint32_t phase = 0;
            for (int t = blockIdx.x; t < p.total_tiles; t += gridDim.x) {
                TileCoord tc = decode_tile(p, t);
                const int nt = p.ntaps[tc.ph], t0 = p.tap0[tc.ph];
                for (int ti = 0; ti < nt; ++ti) {
                    const int x0 = p.stride * tc.gx0 + p.tap_dx[t0 + ti];
                    const int y0 = p.stride * tc.gy0 + p.tap_dy[t0 + ti];
                    const int wt = p.tap_w[t0 + ti];
                    for (int c = 0; c < p.kchunks; ++c) {
                        mbar_wait(&empty_bar[stage], phase ^ 1);
                        uint8_t* st = smem + stage * p.stage_bytes;
                        mbar_arrive_expect_tx(&full_bar[stage], a_bytes * p.split + b_bytes);
                        tma_load_5d(st, &mapA, &full_bar[stage], c * kBK, x0, y0, tc.b, 0);
                        if (p.split == 2)
                            tma_load_5d(st + a_bytes, &mapA, &full_bar[stage], c * kBK, x0, y0, tc.b, 1);
                        tma_load_3d(st + a_bytes * p.split, &mapB, &full_bar[stage], c * kBK,
                                    tc.nt * p.BN, wt);
                        if (++stage == p.stages) { stage = 0; phase ^= 1; }
                    }
                }
            }
        }
    } else if (warp == 1) {
        // ====================== MMA issuer ======================
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            int it = 0;
            for (int t = blockIdx.x; t < p.total_tiles; t += gridDim.x, ++it) {
                TileCoord tc = decode_tile(p, t);
                const int buf = (p.n_accbuf == 2) ? (it & 1) : 0;
                const uint32_t use = (p.n_accbuf == 2) ? (uint32_t)(it >> 1) : (uint32_t)it;
                mbar_wait(&tempty_bar[buf], (use & 1) ^ 1);
                tc_fence_after();
                const uint32_t d = tmem_base + (uint32_t)(buf * p.acc_stride);
                const int nk = p.ntaps[tc.ph] * p.kchunks;
                for (int k = 0; k < nk; ++k) {
                    mbar_wait(&full_bar[stage], phase);
                    tc_fence_after();
                    const uint32_t st = smem_u32(smem + stage * p.stage_bytes);
                    const uint64_t ah = sdesc_sw128(st);
                    const uint64_t al = sdesc_sw128(st + a_bytes);
                    const uint64_t bd = sdesc_sw128(st + a_bytes * p.split);
#pragma unroll
                    for (int kk = 0; kk < kBK / 16; ++kk) {
                        // +32 bytes per 16-element K step inside the 128-byte swizzle row
                        umma_f16(d, ah + 2 * kk, bd + 2 * kk, idesc, (k | kk) != 0);
                        if (p.split == 2) umma_f16(d, al + 2 * kk, bd + 2 * kk, idesc, 1u);
                    }
                    umma_commit(&empty_bar[stage]);
                    if (++stage == p.stages) { stage = 0; phase ^= 1; }
                }
                umma_commit(&tfull_bar[buf]);
            }
        }
    } else if (warp >= 4) {
        // ====================== epilogue ======================
        const int e = threadIdx.x - 128;            // 0..127 = TMEM lane = pixel row of the tile
        const int ew = warp - 4;                    // == warp % 4 -> TMEM lanes 32*ew ..
        const uint32_t lane_off = (uint32_t)(ew * 32) << 16;
        uint32_t norm_phase = 0;
        bool gamma_ready = false;
        int it = 0;
        int sat = 0;
        for (int t = blockIdx.x; t < p.total_tiles; t += gridDim.x, ++it) {
            TileCoord tc = decode_tile(p, t);
            const int buf = (p.n_accbuf == 2) ? (it & 1) : 0;
            const uint32_t use = (p.n_accbuf == 2) ? (uint32_t)(it >> 1) : (uint32_t)it;
            mbar_wait(&tfull_bar[buf], use & 1);
            tc_fence_after();
            const uint32_t dcol = (uint32_t)(buf * p.acc_stride);
            const uint32_t taddr = tmem_base + lane_off + dcol;

            const int gy = tc.gy0 + e / p.Wt, gx = tc.gx0 + e % p.Wt;
            const bool valid = (gy < p.Hg) && (gx < p.Wg);
            const int py = (p.nphase == 4) ? (tc.ph >> 1) : 0;
            const int px = (p.nphase == 4) ? (tc.ph & 1) : 0;
            const int oy = p.out_s * gy + py, ox = p.out_s * gx + px;
            const size_t pix = ((size_t)tc.b * p.Hout + oy) * p.Wout + ox;
            const size_t HWo = (size_t)p.Hout * p.Wout;
            const int co0 = tc.nt * p.BN;

            if (gdn) {
                // ---- norm = x^2 . gamma^T as a second MMA (K = Cout, split hi/lo) ----
                uint8_t* xh = smem + p.off_xsq;
                uint8_t* xl = xh + a_bytes;
                const uint32_t ncol = dcol + (uint32_t)p.BN;     // norm accumulator columns
                for (int c = 0; c < nchunk_out; ++c) {
                    float v[32], hi[32], lo[32];
                    if (c > 0) { mbar_wait(norm_bar, norm_phase); norm_phase ^= 1; }
#pragma unroll
                    for (int half = 0; half < 2; ++half) {
                        __syncwarp();
                        tmem_ld32(taddr + c * 64 + half * 32, v);
#pragma unroll
                        for (int j = 0; j < 32; ++j) {
                            float x = v[j] + __ldg(&p.bias[co0 + c * 64 + half * 32 + j]);
                            float x2 = x * x;
                            __half h = __float2half_rn(x2);
                            hi[j] = __half2float(h);
                            lo[j] = x2 - hi[j];
                        }
                        xsq_store32(xh, e, half * 32, hi);
                        xsq_store32(xl, e, half * 32, lo);
                    }
                    fence_proxy_async_smem();
                    named_bar_sync(1, 128);
                    if (e == 0) {
                        if (!gamma_ready) { mbar_wait(gamma_bar, 0); gamma_ready = true; }
                        tc_fence_after();
                        const uint64_t dh = sdesc_sw128(smem_u32(xh));
                        const uint64_t dl = sdesc_sw128(smem_u32(xl));
                        const uint64_t dg = sdesc_sw128(smem_u32(smem + p.off_gamma + c * b_bytes));
#pragma unroll
                        for (int kk = 0; kk < 4; ++kk) {
                            umma_f16(tmem_base + ncol, dh + 2 * kk, dg + 2 * kk, idesc, (c | kk) != 0);
                            umma_f16(tmem_base + ncol, dl + 2 * kk, dg + 2 * kk, idesc, 1u);
                        }
                        umma_commit(norm_bar);
                    }
                }
                mbar_wait(norm_bar, norm_phase); norm_phase ^= 1;
                tc_fence_after();
                __half* out = reinterpret_cast<__half*>(p.out_act);
                for (int c = 0; c < p.BN / 32; ++c) {
                    float v[32], n[32];
                    __syncwarp();
                    tmem_ld32(taddr + c * 32, v);
                    tmem_ld32(taddr + p.BN + c * 32, n);
                    if (valid) {
#pragma unroll
                        for (int j = 0; j < 32; ++j) {
                            const int co = c * 32 + j;
                            float x = v[j] + __ldg(&p.bias[co]);
                            float nn = __ldg(&p.beta[co]) + n[j];
                            v[j] = (p.ep == EP_GDN) ? x * rsqrtf(nn) : x * sqrtf(nn);
                        }
                        if (p.out_f32) {
#pragma unroll
                            for (int j = 0; j < 32; ++j)
                                p.out_f32[((size_t)tc.b * p.Cout + c * 32 + j) * HWo + (size_t)oy * p.Wout + ox] = v[j];
                        }
                        if (out) {
#pragma unroll
                            for (int q = 0; q < 4; ++q)
                                split_store8(out + pix * p.Cout + c * 32 + q * 8,
                                             p.split == 2 ? out + p.act_plane + pix * p.Cout + c * 32 + q * 8 : nullptr,
                                             v + q * 8);
                        }
                    }
                }
            } else {
                const int ncol32 = (p.BN + 31) / 32;
                for (int c = 0; c < ncol32; ++c) {
                    float v[32];
                    __syncwarp();
                    tmem_ld32(taddr + c * 32, v);
                    const int cb = co0 + c * 32;
                    if (valid && cb < p.Cout) {
                    const int nj = min(32, p.Cout - cb);
#pragma unroll
                    for (int j = 0; j < 32; ++j)
                        if (j < nj) v[j] += __ldg(&p.bias[cb + j]);
                    switch (p.ep) {
                    case EP_F32: {
                        for (int j = 0; j < nj; ++j)
                            p.out_f32[((size_t)tc.b * p.Cout + cb + j) * HWo + (size_t)oy * p.Wout + ox] = v[j];
                        break;
                    }
                    case EP_RELU: {
                        __half* out = reinterpret_cast<__half*>(p.out_act);
#pragma unroll
                        for (int j = 0; j < 32; ++j) v[j] = fmaxf(v[j], 0.0f);
                        if (p.out_f32)
                            for (int j = 0; j < nj; ++j)
                                p.out_f32[((size_t)tc.b * p.Cout + cb + j) * HWo + (size_t)oy * p.Wout + ox] = v[j];
#pragma unroll
                        for (int q = 0; q < 4; ++q)
                            split_store8(out + pix * p.Cout + cb + q * 8,
                                         p.split == 2 ? out + p.act_plane + pix * p.Cout + cb + q * 8 : nullptr,
                                         v + q * 8);
                        break;
                    }
                    case EP_YQUANT:
                    case EP_ZQUANT: {
                        int8_t* sym = reinterpret_cast<int8_t*>(p.out_sym);
                        float av[32];
#pragma unroll
                        for (int j = 0; j < 32; ++j) {
                            float m = (p.mu && j < nj) ? __ldg(&p.mu[cb + j]) : 0.0f;
                            int s = (j < nj) ? round_clamp(v[j] - m, p.L, sat) : 0;
                            if (j < nj) sym[((size_t)tc.b * p.Cout + cb + j) * HWo + (size_t)oy * p.Wout + ox] = (int8_t)s;
                            av[j] = (p.ep == EP_YQUANT) ? fabsf(v[j]) : (float)s + m;
                        }
                        if (p.out_f32)
                            for (int j = 0; j < nj; ++j)
                                p.out_f32[((size_t)tc.b * p.Cout + cb + j) * HWo + (size_t)oy * p.Wout + ox] = v[j];
                        if (p.out_act && (p.ep == EP_ZQUANT || p.abs_out)) {
                            __half* out = reinterpret_cast<__half*>(p.out_act);
#pragma unroll
                            for (int q = 0; q < 4; ++q)
                                split_store8(out + pix * p.Cout + cb + q * 8,
                                             p.split == 2 ? out + p.act_plane + pix * p.Cout + cb + q * 8 : nullptr,
                                             av + q * 8);
                        }
                        break;
                    }
                    case EP_SIGMA: {
                        uint8_t* idx = reinterpret_cast<uint8_t*>(p.out_sym);
                        for (int j = 0; j < nj; ++j) {
                            float s = fmaxf(v[j], 0.0f);
                            if (p.out_f32)
                                p.out_f32[((size_t)tc.b * p.Cout + cb + j) * HWo + (size_t)oy * p.Wout + ox] = s;
                            s = fmaxf(s, 0.11f);
                            // #{ j in [0, 62] : table_j < s } by binary search over the sorted table
                            int lo_i = 0, hi_i = 63;
                            while (lo_i < hi_i) {
                                int mid = (lo_i + hi_i) >> 1;
                                if (__ldg(&p.table[mid]) < s) lo_i = mid + 1; else hi_i = mid;
                            }
                            idx[((size_t)tc.b * p.Cout + cb + j) * HWo + (size_t)oy * p.Wout + ox] = (uint8_t)lo_i;
                        }
                        break;
                    }
                    case EP_FINAL: {
                        const int ry = oy - p.crop_top, rx = ox - p.crop_left;
                        if (ry < 0 || ry >= p.crop_H || rx < 0 || rx >= p.crop_W) break;
                        for (int j = 0; j < nj; ++j) {
                            float xv = fminf(fmaxf(v[j], 0.0f), 1.0f);
                            const int ch = cb + j;
                            if (p.out_f32)
                                p.out_f32[(((size_t)tc.b * p.Cout + ch) * p.crop_H + ry) * p.crop_W + rx] = xv;
                            if (p.out_u8)
                                p.out_u8[(((size_t)tc.b * p.crop_H + ry) * p.crop_W + rx) * 3 + ch] =
                                    (uint8_t)roundf(xv * 255.0f);
                        }
                        break;
                    }
                    default: break;
                    }
                    }
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&tempty_bar[buf]);
        }
        if (p.sat_count) {
            for (int o = 16; o > 0; o >>= 1) sat += __shfl_xor_sync(0xffffffffu, sat, o);
            if (lane == 0 && sat) atomicAdd(p.sat_count, (unsigned long long)sat);
        }
    }

    tc_fence_before();
    __syncthreads();
    if (warp == 2) {
        tc_fence_after();
        tmem_dealloc(tmem_base, (uint32_t)p.tmem_cols);
    }
}

cudaError_t launch_conv_umma(const CUtensorMap& mapA, const CUtensorMap& mapB, const CUtensorMap& mapG,
                             const ConvParams& p, int grid, cudaStream_t stream) {
    static bool attr_set = false;
    if (!attr_set) {
        cudaError_t e = cudaFuncSetAttribute(conv_umma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             227 * 1024);
        if (e != cudaSuccess) return e;
        attr_set = true;
    }
    conv_umma_kernel<<<grid, 256, p.smem_bytes, stream>>>(mapA, mapB, mapG, p);
    return cudaGetLastError();
}

}  // namespace lic
