// aux_kernels.cu -- the small memory-bound kernels around the GEMM engine.
//
//  (frame ingest, step a1, is fused into g_a L1: conv_umma.cu build_l1)
//  sym_ingest    : step a8 (dequantise, "dequantize is exactly symbol +
//                  offset"): int8 CHW symbols -> y-hat / z-hat = s + mu as fp16 hi/lo NHWC.
//  pack_chw      : test export only: f32 CHW -> fp16 hi/lo NHWC.
//  split_reduce  : split-K h layers: the K slices' fp32 partial sums added in slice
//                  order, + bias, then the layer's epilogue exactly as conv_umma.cu applies it
//                  (ReLU -> fp16 hi/lo NHWC; z-quantise -> int8 CHW symbols + z-hat hi/lo NHWC).
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <cstdint>

#include "layer.h"
#include "sigma_index.cuh"

namespace lic {

__device__ __forceinline__ void put_split(__half* out, size_t plane, size_t i, float v, int split) {
    __half h = __float2half_rn(v);
    out[i] = h;
    if (split == 2) out[plane + i] = __float2half_rn(v - __half2float(h));
}

// im2col column k = (ky*5 + kx)*3 + c for k < 75, zero for 75..127

__device__ __forceinline__ uint32_t pack_h2(float a, float b) {
    __half2 h = __floats2half2_rn(a, b);
    return *reinterpret_cast<uint32_t*>(&h);
}

// grid (ceil(W*C/256), H, B): consecutive threads write consecutive NHWC elements
__global__ void __launch_bounds__(256) sym_ingest_kernel(const int8_t* __restrict__ sym, const float* __restrict__ mu,
                                                         int C, int H, int W, __half* __restrict__ out, size_t plane,
                                                         int split) {
    const int i = blockIdx.x * 256 + threadIdx.x;
    if (i >= W * C) return;
    const int x = i / C, c = i - x * C, y = blockIdx.y, b = blockIdx.z;
    const float m = mu ? mu[c] : 0.0f;
    const float v = (float)sym[(((size_t)b * C + c) * H + y) * W + x] + m;
    put_split(out, plane, (((size_t)b * H + y) * W) * C + i, v, split);
}

__global__ void pack_chw_kernel(const float* __restrict__ in, int B, int C, int H, int W,
                                __half* __restrict__ out, size_t plane, int split) {
    const size_t n = (size_t)B * C * H * W;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        const int c = (int)(i % C);
        const size_t pix = i / C;
        const int x = (int)(pix % W);
        const int y = (int)((pix / W) % H);
        const int b = (int)(pix / ((size_t)W * H));
        put_split(out, plane, i, in[(((size_t)b * C + c) * H + y) * W + x], split);
    }
}

// sigma -> index, the same arithmetic as the h_s L3 epilogue (EP_SIGMA in conv_umma.cu)
__global__ void sigma_index_kernel(const float* __restrict__ sigma, size_t n, const float* __restrict__ table,
                                   uint8_t* __restrict__ idx) {
    const auto ltab = [&](int j) { return __ldg(table + j); };
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        idx[i] = (uint8_t)sigma_to_index(sigma[i], ltab);
}

static inline int grid_for(size_t n, int threads) {
    size_t g = (n + threads - 1) / threads;
    return (int)(g > 148 * 16 ? 148 * 16 : (g ? g : 1));
}

// one thread per (pixel, 8 channels); NHWC partials [S][B][H][W][C]
__global__ void __launch_bounds__(256) split_reduce_kernel(
    const float* __restrict__ part, int S, int B, int H, int W, int C, const float* __restrict__ bias,
    const float* __restrict__ mu, int ep, int L, __half* __restrict__ out_act, size_t act_plane, int split,
    int8_t* __restrict__ out_sym, float* __restrict__ out_f32, unsigned long long* sat_count,
    unsigned long long* range_count) {
    const size_t n8 = (size_t)B * H * W * (C / 8);
    const size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    int sat = 0, ovf = 0;
    if (i < n8) {
        const size_t pix = i / (C / 8);
        const int c0 = (int)(i - pix * (C / 8)) * 8;
        const size_t stride = (size_t)B * H * W * C;
        const float4* src = reinterpret_cast<const float4*>(part + pix * C + c0);
        float4 a = src[0], b = src[1];
        for (int s = 1; s < S; ++s) {                      // slice order: deterministic
            const float4* q = reinterpret_cast<const float4*>(part + s * stride + pix * C + c0);
            const float4 qa = q[0], qb = q[1];
            a.x += qa.x; a.y += qa.y; a.z += qa.z; a.w += qa.w;
            b.x += qb.x; b.y += qb.y; b.z += qb.z; b.w += qb.w;
        }
        float v[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
#pragma unroll
        for (int j = 0; j < 8; ++j) v[j] += bias[c0 + j];
        const int bb = (int)(pix / ((size_t)H * W));
        const size_t rem = pix - (size_t)bb * H * W;
        const size_t HW = (size_t)H * W;
        const size_t chw0 = (size_t)bb * C * HW + rem;     // + channel * HW
        float o[8];
        if (ep == EP_ZQUANT) {
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const float m = mu ? mu[c0 + j] : 0.0f;
                float r = roundf(v[j] - m);                // half away from zero (R4)
                if (r > (float)L) { r = (float)L; ++sat; }
                if (r < (float)-L) { r = (float)-L; ++sat; }
                if (out_sym) out_sym[chw0 + (size_t)(c0 + j) * HW] = (int8_t)(int)r;
                o[j] = r + m;
            }
        } else {                                           // EP_RELU
#pragma unroll
            for (int j = 0; j < 8; ++j) { v[j] = fmaxf(v[j], 0.0f); o[j] = v[j]; }
        }
        if (out_f32) {
#pragma unroll
            for (int j = 0; j < 8; ++j) out_f32[chw0 + (size_t)(c0 + j) * HW] = v[j];
        }
        if (out_act) {
            // the fp16 range guard of the GEMM epilogue (R16d), then hi / lo planes
#pragma unroll
            for (int j = 0; j < 8; ++j)
                if (fabsf(o[j]) > 65504.0f) { ++ovf; o[j] = copysignf(65504.0f, o[j]); }
            uint4 h, l;
            uint32_t* hp = &h.x;
            uint32_t* lp = &l.x;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const __half2 hh = __floats2half2_rn(o[2 * k], o[2 * k + 1]);
                const float2 hf = __half22float2(hh);
                hp[k] = *reinterpret_cast<const uint32_t*>(&hh);
                lp[k] = pack_h2(o[2 * k] - hf.x, o[2 * k + 1] - hf.y);
            }
            *reinterpret_cast<uint4*>(out_act + pix * C + c0) = h;
            if (split == 2) *reinterpret_cast<uint4*>(out_act + act_plane + pix * C + c0) = l;
        }
    }
    for (int o2 = 16; o2 > 0; o2 >>= 1) {
        sat += __shfl_xor_sync(0xffffffffu, sat, o2);
        ovf += __shfl_xor_sync(0xffffffffu, ovf, o2);
    }
    if ((threadIdx.x & 31) == 0) {
        if (sat && sat_count) atomicAdd(sat_count, (unsigned long long)sat);
        if (ovf && range_count) atomicAdd(range_count, (unsigned long long)ovf);
    }
}

cudaError_t launch_split_reduce(const float* part, int S, int B, int H, int W, int C, const float* bias,
                                const float* mu, int ep, int L, __half* out_act, size_t act_plane, int split,
                                int8_t* out_sym, float* out_f32, unsigned long long* sat_count,
                                unsigned long long* range_count, cudaStream_t st) {
    const size_t n8 = (size_t)B * H * W * (C / 8);
    const unsigned grid = (unsigned)((n8 + 255) / 256);
    split_reduce_kernel<<<grid, 256, 0, st>>>(part, S, B, H, W, C, bias, mu, ep, L, out_act, act_plane, split, out_sym,
                                               out_f32, sat_count, range_count);
    return cudaGetLastError();
}

cudaError_t launch_sym_ingest(const int8_t* sym, const float* mu, int B, int C, int H, int W, __half* out,
                              size_t plane, int split, cudaStream_t st) {
    const dim3 grid((W * C + 255) / 256, H, B);
    sym_ingest_kernel<<<grid, 256, 0, st>>>(sym, mu, C, H, W, out, plane, split);
    return cudaGetLastError();
}

cudaError_t launch_pack_chw(const float* in, int B, int C, int H, int W, __half* out, size_t plane, int split,
                            cudaStream_t st) {
    const size_t n = (size_t)B * C * H * W;
    pack_chw_kernel<<<grid_for(n, 256), 256, 0, st>>>(in, B, C, H, W, out, plane, split);
    return cudaGetLastError();
}

cudaError_t launch_sigma_index(const float* sigma, size_t n, const float* table, uint8_t* idx, cudaStream_t st) {
    sigma_index_kernel<<<grid_for(n, 256), 256, 0, st>>>(sigma, n, table, idx);
    return cudaGetLastError();
}

}  // namespace lic
