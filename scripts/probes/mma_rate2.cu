// mma_rate2.cu -- what slows the engine's MMAs below the pure tcgen05 rate?  M = 128, N = 128,
// K = 16 (64 cycles each when issued back to back).  Variants:
//   0: back to back (8 per group, commit per group, no waits)
//   1: + per group an mbarrier try_wait on an already-completed barrier and a fence (the MMA
//      warp's bookkeeping)
//   2: + 8 other warps streaming st.shared / ld.shared (epilogue staging traffic, ~64 B/clk)
//   3: + one warp issuing TMA-like bulk smem writes (cp.async.bulk global->shared, 8 KB each)
//   4: variant 1 without the try_wait (fence only);  5: variant 1 without the fence (try_wait only)
#include <cstdio>
#include <cuda_fp16.h>
#include "../../paper_2208_01641_b200/csrc/ptx.cuh"
using namespace lic;

__device__ __forceinline__ void stsu4(uint32_t addr, uint4 v) {
    asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" :: "r"(addr), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
                 : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 :: "r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}

__global__ void rate(long long* out, int iters, int variant, const uint8_t* gsrc) {
    extern __shared__ __align__(1024) uint8_t sm[];
    uint8_t* smem = (uint8_t*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
    __shared__ uint64_t bar, done_bar, tbar;
    __shared__ uint32_t slot;
    __shared__ volatile int stop;
    for (int i = threadIdx.x; i < (128 * 128 + 128 * 128) / 16; i += blockDim.x) ((uint4*)smem)[i] = make_uint4(0x3c003c00u, 0, 0, 0);
    fence_proxy_async_smem();
    if (threadIdx.x == 0) { mbar_init(&bar, 1); mbar_init(&done_bar, 1); mbar_init(&tbar, 1); stop = 0; fence_mbar_init(); }
    if (threadIdx.x < 32) tmem_alloc(&slot, 256);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tm = slot;
    const int warp = threadIdx.x >> 5;
    if (warp == 0) {
        if (threadIdx.x == 0) mbar_arrive(&done_bar);            // completes phase 0 immediately
        __syncwarp();
        const uint64_t ad = sdesc_sw128(smem_u32(smem));
        const uint64_t bd = sdesc_sw128(smem_u32(smem + 128 * 128));
        const long long t0 = clock64();
        bool nxt_ready = true;
        for (int it = 0; it < iters; ++it) {
            if (variant == 6) {
                // the next group's barrier tested before this group's MMAs (latency overlapped)
                if (!nxt_ready) { while (!mbar_test(&done_bar, 0)) {} }
                tc_fence_after();
            }
            if (variant >= 1 && variant != 4 && variant != 6) { while (!mbar_test(&done_bar, 0)) {} }
            if (variant >= 1 && variant != 5 && variant != 6) tc_fence_after();
            if (variant == 6) nxt_ready = mbar_test(&done_bar, 0);
            if (variant == 8) {
                if (threadIdx.x == 0) {
#pragma unroll
                    for (int kk = 0; kk < 8; ++kk) umma_f16(tm, ad + 2 * (kk & 3), bd + 2 * (kk & 3), idesc_f16_f32(128, 128), (it | kk) != 0);
                    umma_commit(&bar);
                }
            } else if (elect_one()) {
#pragma unroll
                for (int kk = 0; kk < 8; ++kk) umma_f16(tm, ad + 2 * (kk & 3), bd + 2 * (kk & 3), idesc_f16_f32(128, 128), (it | kk) != 0);
                if (variant != 7 || it == iters - 1) umma_commit(&bar);
            }
            if (variant != 8) __syncwarp();
        }
        if (threadIdx.x == 0) {
            mbar_wait(&bar, variant == 7 ? 0 : ((iters - 1) & 1));
            const long long t1 = clock64();
            if (blockIdx.x == 0) out[0] = t1 - t0;
            stop = 1;
        }
        __syncwarp();
    } else if (variant >= 2 && variant <= 3 && warp >= 4 && warp < 12) {
        uint8_t* buf = smem + 64 * 1024 + (warp - 4) * 4096;
        uint4 v = make_uint4(threadIdx.x, 1, 2, 3);
        while (!stop) {
            for (int k = 0; k < 8; ++k) {
                stsu4(smem_u32(buf) + (uint32_t)(((k * 32 + (threadIdx.x & 31)) * 16) & 4095), v);
                v.x += 1;
            }
            __syncwarp();
        }
    } else if (variant == 3 && warp == 1) {
        uint32_t ph = 0;
        while (!stop) {
            if (threadIdx.x == 32) {
                mbar_arrive_expect_tx(&tbar, 8192);
                bulk_g2s(smem + 100 * 1024, gsrc + (blockIdx.x & 63) * 8192, 8192, &tbar);
            }
            __syncwarp();
            mbar_wait(&tbar, ph);
            ph ^= 1;
        }
    }
    tc_fence_before();
    __syncthreads();
    if (threadIdx.x < 32) { tc_fence_after(); tmem_dealloc(tm, 256); }
}

int main() {
    long long* d;
    uint8_t* g;
    cudaMalloc(&d, 8);
    cudaMalloc(&g, 1 << 20);
    const int iters = 1000;
    cudaFuncSetAttribute(rate, cudaFuncAttributeMaxDynamicSharedMemorySize, 120 * 1024);
    for (int v = 0; v < 9; ++v) {
        rate<<<148, 384, 120 * 1024>>>(d, iters, v, g);
        cudaDeviceSynchronize();
        rate<<<148, 384, 120 * 1024>>>(d, iters, v, g);
        cudaError_t e = cudaDeviceSynchronize();
        long long c = 0;
        cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
        printf("variant %d: %.1f cycles per MMA %s\n", v, (double)c / (iters * 8), e == cudaSuccess ? "" : cudaGetErrorString(e));
    }
    return 0;
}
