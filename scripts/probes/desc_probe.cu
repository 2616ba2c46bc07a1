// desc_probe.cu -- does a tcgen05 K-major SW128 smem descriptor accept a start address that
// is not 1024-byte aligned (row offset s0 inside the swizzle atom) and an SBO that is not a
// multiple of 1024 (8-row groups at arbitrary row stride)?  Answers whether shifted windows
// of a resident halo tile can be fed to the MMA directly.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_fp16.h>
#include "../../paper_2208_01641_b200/csrc/ptx.cuh"
using namespace lic;

__device__ uint64_t desc_custom(uint32_t start, uint32_t sbo_bytes, uint32_t base_off) {
    uint64_t d = 0;
    d |= (uint64_t)((start >> 4) & 0x3FFF);
    d |= (uint64_t)((sbo_bytes >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;
    d |= (uint64_t)(base_off & 7) << 49;
    d |= (uint64_t)2 << 61;
    return d;
}

__global__ void probe(const __half* A, int arows, const __half* Bm, float* D, int s0, int sbo_rows, int boff_mode) {
    extern __shared__ __align__(1024) uint8_t sm[];
    uint8_t* smem = (uint8_t*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
    uint8_t* sa = smem;
    uint8_t* sb = smem + ((arows * 128 + 1023) / 1024) * 1024;
    __shared__ uint64_t bar;
    __shared__ uint32_t slot;
    for (int i = threadIdx.x; i < arows * 8; i += blockDim.x) {
        int r = i / 8, j = i % 8;
        *(uint4*)(sa + r * 128 + ((j ^ (r & 7)) * 16)) = *(const uint4*)(A + r * 64 + j * 8);
    }
    for (int i = threadIdx.x; i < 16 * 8; i += blockDim.x) {
        int r = i / 8, j = i % 8;
        *(uint4*)(sb + r * 128 + ((j ^ (r & 7)) * 16)) = *(const uint4*)(Bm + r * 64 + j * 8);
    }
    fence_proxy_async_smem();
    if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
    if (threadIdx.x < 32) tmem_alloc(&slot, 32);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tm = slot;
    if (threadIdx.x == 0) {
        const uint32_t start = smem_u32(sa) + s0 * 128;
        const uint32_t boff = boff_mode == 1 ? ((start >> 7) & 7) : 0;
        const uint64_t ad = desc_custom(start, sbo_rows * 128, boff);
        const uint64_t bd = sdesc_sw128(smem_u32(sb));
        for (int kk = 0; kk < 4; ++kk) umma_f16(tm, ad + 2 * kk, bd + 2 * kk, idesc_f16_f32(128, 16), kk > 0);
        umma_commit(&bar);
    }
    mbar_wait(&bar, 0);
    tc_fence_after();
    float v[16];
    const int w = threadIdx.x / 32;
    tmem_ld16(tm + ((uint32_t)(w * 32) << 16), v);
    for (int j = 0; j < 16; ++j) D[threadIdx.x * 16 + j] = v[j];
    tc_fence_before();
    __syncthreads();
    if (threadIdx.x < 32) { tc_fence_after(); tmem_dealloc(tm, 32); }
}

int main() {
    const int arows = 256;
    std::vector<__half> A(arows * 64), B(16 * 64);
    std::vector<float> Af(arows * 64), Bf(16 * 64);
    srand(1);
    for (int i = 0; i < arows * 64; ++i) { int v = rand() % 5 - 2; Af[i] = v; A[i] = __float2half((float)v); }
    for (int i = 0; i < 16 * 64; ++i) { int v = rand() % 5 - 2; Bf[i] = v; B[i] = __float2half((float)v); }
    __half *dA, *dB; float* dD;
    cudaMalloc(&dA, A.size() * 2); cudaMalloc(&dB, B.size() * 2); cudaMalloc(&dD, 128 * 16 * 4);
    cudaMemcpy(dA, A.data(), A.size() * 2, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, B.data(), B.size() * 2, cudaMemcpyHostToDevice);
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
    const int s0s[] = {0, 1, 3, 5, 8, 11, 13, 21};
    const int sbos[] = {8, 10, 18};
    for (int sbo : sbos)
        for (int s0 : s0s)
            for (int bm = 0; bm < 2; ++bm) {
                probe<<<1, 128, 100 * 1024>>>(dA, arows, dB, dD, s0, sbo, bm);
                cudaError_t e = cudaDeviceSynchronize();
                if (e != cudaSuccess) { printf("sbo %d s0 %d boff %d: CUDA error %s\n", sbo, s0, bm, cudaGetErrorString(e)); return 1; }
                std::vector<float> Dh(128 * 16);
                cudaMemcpy(Dh.data(), dD, Dh.size() * 4, cudaMemcpyDeviceToHost);
                double maxerr = 0;
                for (int m = 0; m < 128; ++m) {
                    const int row = s0 + (m / 8) * sbo + (m % 8);
                    for (int n = 0; n < 16; ++n) {
                        float ref = 0;
                        for (int k = 0; k < 64; ++k) ref += Af[row * 64 + k] * Bf[n * 64 + k];
                        maxerr = std::max(maxerr, (double)std::abs(ref - Dh[m * 16 + n]));
                    }
                }
                printf("sbo_rows %2d s0 %2d base_offset %s: max err %g %s\n", sbo, s0, bm ? "(start>>7)&7" : "0         ",
                       maxerr, maxerr == 0 ? "OK" : "MISMATCH");
            }
    return 0;
}
