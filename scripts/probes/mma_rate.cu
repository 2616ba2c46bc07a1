// mma_rate.cu -- back-to-back tcgen05.mma kind::f16 (cta_group::1, M = 128, K = 16) from smem
// operands with nothing else running: cycles per MMA for N = 64 / 128 / 256, one CTA per SM on
// all SMs.  Tells whether the engine's ~90 cycles per M256xN128 pair MMA is the hardware rate.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o mma_rate scripts/probes/mma_rate.cu
#include <cstdio>
#include <cuda_fp16.h>
#include "../../paper_2208_01641_b200/csrc/ptx.cuh"
using namespace lic;

template <int N>
__global__ void rate(long long* out, int iters) {
    extern __shared__ __align__(1024) uint8_t sm[];
    uint8_t* smem = (uint8_t*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
    __shared__ uint64_t bar;
    __shared__ uint32_t slot;
    for (int i = threadIdx.x; i < (128 * 128 + N * 128) / 16; i += blockDim.x) ((uint4*)smem)[i] = make_uint4(0x3c003c00u, 0, 0, 0);
    fence_proxy_async_smem();
    if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
    if (threadIdx.x < 32) tmem_alloc(&slot, 256);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tm = slot;
    if (threadIdx.x == 0) {
        const uint64_t ad = sdesc_sw128(smem_u32(smem));
        const uint64_t bd = sdesc_sw128(smem_u32(smem + 128 * 128));
        const long long t0 = clock64();
        for (int it = 0; it < iters; ++it)
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) umma_f16(tm, ad + 2 * kk, bd + 2 * kk, idesc_f16_f32(128, N), (it | kk) != 0);
        umma_commit(&bar);
        mbar_wait(&bar, 0);
        const long long t1 = clock64();
        if (blockIdx.x == 0) out[0] = t1 - t0;
    }
    tc_fence_before();
    __syncthreads();
    if (threadIdx.x < 32) { tc_fence_after(); tmem_dealloc(tm, 256); }
}

int main() {
    long long* d;
    cudaMalloc(&d, 8);
    const int iters = 2000;
    auto run = [&](auto kern, int n) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 120 * 1024);
        kern<<<148, 128, 120 * 1024>>>(d, iters);
        cudaDeviceSynchronize();
        kern<<<148, 128, 120 * 1024>>>(d, iters);
        cudaError_t e = cudaDeviceSynchronize();
        long long c = 0;
        cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
        printf("M=128 N=%d K=16: %.1f cycles per MMA (nominal %d) %s\n", n, (double)c / (iters * 4), n / 2,
               e == cudaSuccess ? "" : cudaGetErrorString(e));
    };
    run(rate<64>, 64);
    run(rate<128>, 128);
    run(rate<256>, 256);
    return 0;
}
