// aux_kernels.cu -- the small memory-bound kernels around the GEMM engine.
//
//  (frame ingest, step a1, is fused into g_a L1: conv_umma.cu build_l1)
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
