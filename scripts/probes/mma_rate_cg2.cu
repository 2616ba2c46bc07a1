// mma_rate_cg2.cu -- back-to-back tcgen05.mma.cta_group::2 (M = 256 over a CTA pair, N = 128,
// K = 16), issued by the leader CTA: cycles per MMA (compare mma_rate.cu's cta_group::1 64).
#include <cstdio>
#include <cuda_fp16.h>
#include "../../paper_2208_01641_b200/csrc/ptx.cuh"
using namespace lic;

__global__ void __cluster_dims__(2, 1, 1) rate(long long* out, int iters, int groups_wait) {
    extern __shared__ __align__(1024) uint8_t sm[];
    uint8_t* smem = (uint8_t*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
    __shared__ uint64_t bar, done_bar;
    __shared__ uint32_t slot;
    for (int i = threadIdx.x; i < (128 * 128 + 64 * 128) / 16; i += blockDim.x) ((uint4*)smem)[i] = make_uint4(0x3c003c00u, 0, 0, 0);
    fence_proxy_async_smem();
    if (threadIdx.x == 0) { mbar_init(&bar, 1); mbar_init(&done_bar, 1); fence_mbar_init(); }
    if (threadIdx.x < 32) tmem_alloc_cg2(&slot, 256);
    tc_fence_before();
    cluster_sync_all();
    tc_fence_after();
    const uint32_t tm = slot;
    const bool leader = cluster_ctarank() == 0;
    if (threadIdx.x == 0 && leader) {
        mbar_arrive(&done_bar);
        const uint64_t ad = sdesc_sw128(smem_u32(smem));
        const uint64_t bd = sdesc_sw128(smem_u32(smem + 128 * 128));
        const uint32_t id = idesc_f16_f32(256, 128);
        const long long t0 = clock64();
        for (int it = 0; it < iters; ++it) {
            if (groups_wait) { while (!mbar_test(&done_bar, 0)) {} tc_fence_after(); }
#pragma unroll
            for (int kk = 0; kk < 8; ++kk) umma_f16_cg2(tm, ad + 2 * (kk & 3), bd + 2 * (kk & 3), id, (it | kk) != 0);
            umma_commit_pair(&bar);
        }
        while (!mbar_test(&bar, 0) && !mbar_test(&bar, 1)) {}
        const long long t1 = clock64();
        if (blockIdx.x == 0) out[0] = t1 - t0;
    }
    tc_fence_before();
    cluster_sync_all();
    if (threadIdx.x < 32) { tc_fence_after(); tmem_dealloc_cg2(tm, 256); }
}

int main() {
    long long* d;
    cudaMalloc(&d, 8);
    const int iters = 2000;
    cudaFuncSetAttribute(rate, cudaFuncAttributeMaxDynamicSharedMemorySize, 80 * 1024);
    for (int w = 0; w < 2; ++w) {
        rate<<<148, 128, 80 * 1024>>>(d, iters, w);
        cudaDeviceSynchronize();
        rate<<<148, 128, 80 * 1024>>>(d, iters, w);
        cudaError_t e = cudaDeviceSynchronize();
        long long c = 0;
        cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
        printf("cta_group::2 M=256 N=128 K=16%s: %.1f cycles per MMA %s\n", w ? " + wait/fence per 8" : "",
               (double)c / (iters * 8), e == cudaSuccess ? "" : cudaGetErrorString(e));
    }
    return 0;
}
