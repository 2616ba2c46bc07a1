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

// one thread per (output pixel, k); k = (ky*5 + kx)*3 + c for k < 75, zero for 75..127
template <typename T>
__global__ void ingest_im2col_kernel(const T* __restrict__ fr, int hwc, int B, int H, int W, int top,
                                     int left, int Ho, int Wo, __half* __restrict__ out, size_t plane,
                                     int split) {
    const size_t n = (size_t)B * Ho * Wo * 128;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        const int k = (int)(i & 127);
        const size_t pix = i >> 7;
        const int ox = (int)(pix % Wo);
        const int oy = (int)((pix / Wo) % Ho);
        const int b = (int)(pix / ((size_t)Wo * Ho));
        float v = 0.0f;
        if (k < 75) {
            const int ky = k / 15, r = k % 15, kx = r / 3, c = r % 3;
            const int iy = 2 * oy + ky - 2 - top, ix = 2 * ox + kx - 2 - left;
            if (iy >= 0 && iy < H && ix >= 0 && ix < W) {
                if (hwc) v = (float)fr[(((size_t)b * H + iy) * W + ix) * 3 + c] / 255.0f;  // u8 / 255
                else v = (float)fr[(((size_t)b * 3 + c) * H + iy) * W + ix];
            }
        }
        put_split(out, plane, i, v, split);
    }
}

__global__ void sym_ingest_kernel(const int8_t* __restrict__ sym, const float* __restrict__ mu, int B, int C,
                                  int H, int W, __half* __restrict__ out, size_t plane, int split) {
    const size_t n = (size_t)B * C * H * W;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        // i enumerates NHWC output order: coalesced writes
        const int c = (int)(i % C);
        const size_t pix = i / C;
        const int x = (int)(pix % W);
        const int y = (int)((pix / W) % H);
        const int b = (int)(pix / ((size_t)W * H));
        const float m = mu ? mu[c] : 0.0f;
        const float v = (float)sym[(((size_t)b * C + c) * H + y) * W + x] + m;
        put_split(out, plane, i, v, split);
    }
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
    const size_t n = (size_t)B * Ho * Wo * 128;
    if (hwc)
        ingest_im2col_kernel<uint8_t><<<grid_for(n, 256), 256, 0, st>>>(
            (const uint8_t*)fr, 1, B, H, W, top, left, Ho, Wo, out, plane, split);
    else
        ingest_im2col_kernel<float><<<grid_for(n, 256), 256, 0, st>>>(
            (const float*)fr, 0, B, H, W, top, left, Ho, Wo, out, plane, split);
    return cudaGetLastError();
}

cudaError_t launch_sym_ingest(const int8_t* sym, const float* mu, int B, int C, int H, int W, __half* out,
                              size_t plane, int split, cudaStream_t st) {
    const size_t n = (size_t)B * C * H * W;
    sym_ingest_kernel<<<grid_for(n, 256), 256, 0, st>>>(sym, mu, B, C, H, W, out, plane, split);
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
