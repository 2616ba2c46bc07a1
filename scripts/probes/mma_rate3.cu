// mma_rate3.cu -- cost of the per-group bookkeeping of an MMA issuer, compile-time variants, one
// thread issuing groups of 8 tcgen05.mma (M = 128, N = 128, K = 16; 64 cycles each back to back):
//   A: nothing between groups          B: a commit per group
//   C: try_wait (completed) per group  D: commit + try_wait + fence per group
//   E: D with the next group's try_wait issued before this group's MMAs
#include <cstdio>
#include <cuda_fp16.h>
#include "../../paper_2208_01641_b200/csrc/ptx.cuh"
using namespace lic;

template <int V>
__global__ void rate(long long* out, int iters) {
    extern __shared__ __align__(1024) uint8_t sm[];
    uint8_t* smem = (uint8_t*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
    __shared__ uint64_t bar, done_bar;
    __shared__ uint32_t slot;
    for (int i = threadIdx.x; i < (128 * 128 * 2) / 16; i += blockDim.x) ((uint4*)smem)[i] = make_uint4(0x3c003c00u, 0, 0, 0);
    fence_proxy_async_smem();
    if (threadIdx.x == 0) { mbar_init(&bar, 1); mbar_init(&done_bar, 1); fence_mbar_init(); }
    if (threadIdx.x < 32) tmem_alloc(&slot, 256);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tm = slot;
    if (threadIdx.x == 0) {
        mbar_arrive(&done_bar);
        const uint64_t ad = sdesc_sw128(smem_u32(smem));
        const uint64_t bd = sdesc_sw128(smem_u32(smem + 128 * 128));
        const uint32_t id = idesc_f16_f32(128, 128);
        const long long t0 = clock64();
        bool ready = mbar_test(&done_bar, 0);
        for (int it = 0; it < iters; ++it) {
            if (V == 2 || V == 3) { while (!mbar_test(&done_bar, 0)) {} }
            if (V == 4) { while (!ready) ready = mbar_test(&done_bar, 0); }
            if (V >= 3) tc_fence_after();
            if (V == 4) ready = mbar_test(&done_bar, 0);
#pragma unroll
            for (int kk = 0; kk < 8; ++kk) umma_f16(tm, ad + 2 * (kk & 3), bd + 2 * (kk & 3), id, (it | kk) != 0);
            if (V == 1 || V >= 3) umma_commit(&bar);
        }
        umma_commit(&bar);
        while (!mbar_test(&bar, 0) && !mbar_test(&bar, 1)) {}
        const long long t1 = clock64();
        if (blockIdx.x == 0) out[0] = t1 - t0;
    }
    tc_fence_before();
    __syncthreads();
    if (threadIdx.x < 32) { tc_fence_after(); tmem_dealloc(tm, 256); }
}

template <int V>
void run(long long* d, const char* name) {
    const int iters = 2000;
    cudaFuncSetAttribute(rate<V>, cudaFuncAttributeMaxDynamicSharedMemorySize, 80 * 1024);
    rate<V><<<148, 128, 80 * 1024>>>(d, iters);
    cudaDeviceSynchronize();
    rate<V><<<148, 128, 80 * 1024>>>(d, iters);
    cudaError_t e = cudaDeviceSynchronize();
    long long c = 0;
    cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
    printf("%s: %.1f cycles per MMA %s\n", name, (double)c / (iters * 8), e == cudaSuccess ? "" : cudaGetErrorString(e));
}

int main() {
    long long* d;
    cudaMalloc(&d, 8);
    run<0>(d, "A nothing");
    run<1>(d, "B commit/group");
    run<2>(d, "C try_wait/group");
    run<3>(d, "D commit+try_wait+fence");
    run<4>(d, "E D with early try_wait");
    return 0;
}
