// aux_kernels.cu -- the small memory-bound kernels around the GEMM engine.
//
//  ingest_im2col : step a1 (frame ingest + centred zero pad, SURVEY.md §8(c) step 1:
//                  x = u8/255 or f32 as given) fused with the im2col of g_a L1
//                  (conv 5x5/s2, Cin = 3, K = 75 padded to 128), written as fp16 hi/lo
//                  NHWC-128 rows so L1 runs as a plain GEMM on the same tcgen05 engine.
//  sym_ingest    : step a8 (dequantise, "dequantize is exactly symbol +
//                  offset"): int8 CHW symbols -> y-hat / z-hat = s + mu as fp16 hi/lo NHWC.
//  pack_chw      : test export only: f32 CHW -> fp16 hi/lo NHWC.
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <cstdint>

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

// grid (ceil(Wo/128), Ho, B), 128 threads: one thread per output pixel builds its 75 im2col
// values (25 taps x RGB) and writes its 128-column hi and lo rows (256 B each, 16-byte stores)
template <typename T>
__global__ void __launch_bounds__(128) ingest_im2col_kernel(const T* __restrict__ fr, int hwc, int H, int W,
                                                            int top, int left, int Ho, int Wo,
                                                            __half* __restrict__ out, size_t plane, int split) {
    // x = u8 / 255 (IEEE fp32 division) tabulated once per block
    __shared__ float s_u8[256];
    for (int v = threadIdx.x; v < 256; v += blockDim.x) s_u8[v] = __fdiv_rn((float)v, 255.0f);
    __syncthreads();
    const int ox = blockIdx.x * 128 + threadIdx.x, oy = blockIdx.y, b = blockIdx.z;
    if (ox >= Wo) return;
    float v[80];
#pragma unroll
    for (int ky = 0; ky < 5; ++ky) {
        const int iy = 2 * oy + ky - 2 - top;
        const bool rowok = iy >= 0 && iy < H;
#pragma unroll
        for (int kx = 0; kx < 5; ++kx) {
            const int ix = 2 * ox + kx - 2 - left;
            const bool ok = rowok && ix >= 0 && ix < W;
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                float val = 0.0f;
                if (ok) {
                    if (hwc) val = s_u8[(int)fr[(((size_t)b * H + iy) * W + ix) * 3 + c]];
                    else val = (float)fr[(((size_t)b * 3 + c) * H + iy) * W + ix];
                }
                v[(ky * 5 + kx) * 3 + c] = val;
            }
        }
    }
#pragma unroll
    for (int k = 75; k < 80; ++k) v[k] = 0.0f;
    uint4* oh = reinterpret_cast<uint4*>(out + (((size_t)b * Ho + oy) * Wo + ox) * 128);
    uint4* ol = reinterpret_cast<uint4*>(out + plane + (((size_t)b * Ho + oy) * Wo + ox) * 128);
#pragma unroll
    for (int g = 0; g < 10; ++g) {
        const float* w = v + 8 * g;
        uint4 hi, lo;
        hi.x = pack_h2(w[0], w[1]); hi.y = pack_h2(w[2], w[3]); hi.z = pack_h2(w[4], w[5]); hi.w = pack_h2(w[6], w[7]);
        lo.x = pack_h2(w[0] - __half2float(__float2half_rn(w[0])), w[1] - __half2float(__float2half_rn(w[1])));
        lo.y = pack_h2(w[2] - __half2float(__float2half_rn(w[2])), w[3] - __half2float(__float2half_rn(w[3])));
        lo.z = pack_h2(w[4] - __half2float(__float2half_rn(w[4])), w[5] - __half2float(__float2half_rn(w[5])));
        lo.w = pack_h2(w[6] - __half2float(__float2half_rn(w[6])), w[7] - __half2float(__float2half_rn(w[7])));
        oh[g] = hi;
        if (split == 2) ol[g] = lo;
    }
    const uint4 z = make_uint4(0, 0, 0, 0);
#pragma unroll
    for (int g = 10; g < 16; ++g) {
        oh[g] = z;
        if (split == 2) ol[g] = z;
    }
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
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        const float s = fmaxf(sigma[i], 0.11f);
        int lo = 0, hi = 63;
        while (lo < hi) {
            int mid = (lo + hi) >> 1;
            if (table[mid] < s) lo = mid + 1; else hi = mid;
        }
        idx[i] = (uint8_t)lo;
    }
}

static inline int grid_for(size_t n, int threads) {
    size_t g = (n + threads - 1) / threads;
    return (int)(g > 148 * 16 ? 148 * 16 : (g ? g : 1));
}

cudaError_t launch_ingest(const void* fr, int hwc, int B, int H, int W, int top, int left, int Ho, int Wo,
                          __half* out, size_t plane, int split, cudaStream_t st) {
    const dim3 grid((Wo + 127) / 128, Ho, B);
    if (hwc)
        ingest_im2col_kernel<uint8_t><<<grid, 128, 0, st>>>((const uint8_t*)fr, 1, H, W, top, left, Ho, Wo, out,
                                                            plane, split);
    else
        ingest_im2col_kernel<float><<<grid, 128, 0, st>>>((const float*)fr, 0, H, W, top, left, Ho, Wo, out, plane,
                                                          split);
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
