// f8_probe.cu -- tcgen05.mma kind::f8f6f4 with e4m3 A and B, K-major SW128 smem (128-byte rows
// = 128 K elements), K = 32 per instruction (+32 B per step): does D = A . B^T come out right,
// with the kind::f16 instruction descriptor (A/B format 0 = E4M3)?  Also checks
// cvt.rn.satfinite.e4m3x2.f32 on the device.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o f8_probe scripts/probes/f8_probe.cu
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>
#include <cuda_fp8.h>
#include <cuda_fp16.h>
#include "../../paper_2208_01641_b200/csrc/ptx.cuh"
using namespace lic;

__device__ __forceinline__ void umma_f8(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                        uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f8f6f4 [%0], %1, %2, %3, p;\n\t}"
        :: "r"(d_tmem), "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate) : "memory");
}

__global__ void probe(const uint8_t* A, const uint8_t* Bm, float* D, float* cvt_out, const float* cvt_in) {
    extern __shared__ __align__(1024) uint8_t sm[];
    uint8_t* smem = (uint8_t*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
    uint8_t* sa = smem;                 // 128 rows x 128 B
    uint8_t* sb = smem + 128 * 128;     // 16 rows x 128 B
    __shared__ uint64_t bar;
    __shared__ uint32_t slot;
    for (int i = threadIdx.x; i < 128 * 8; i += blockDim.x) {
        int r = i / 8, j = i % 8;
        *(uint4*)(sa + r * 128 + ((j ^ (r & 7)) * 16)) = *(const uint4*)(A + r * 128 + j * 16);
    }
    for (int i = threadIdx.x; i < 16 * 8; i += blockDim.x) {
        int r = i / 8, j = i % 8;
        *(uint4*)(sb + r * 128 + ((j ^ (r & 7)) * 16)) = *(const uint4*)(Bm + r * 128 + j * 16);
    }
    // device conversion check: pairs -> e4m3x2 -> back
    if (threadIdx.x < 64) {
        __nv_fp8x2_e4m3 p(make_float2(cvt_in[2 * threadIdx.x], cvt_in[2 * threadIdx.x + 1]));
        float2 b = float2(p);
        cvt_out[2 * threadIdx.x] = b.x;
        cvt_out[2 * threadIdx.x + 1] = b.y;
    }
    fence_proxy_async_smem();
    if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
    if (threadIdx.x < 32) tmem_alloc(&slot, 32);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tm = slot;
    if (threadIdx.x == 0) {
        const uint64_t ad = sdesc_sw128(smem_u32(sa));
        const uint64_t bd = sdesc_sw128(smem_u32(sb));
        for (int kk = 0; kk < 4; ++kk) umma_f8(tm, ad + 2 * kk, bd + 2 * kk, idesc_f16_f32(128, 16), kk > 0);
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

static float e4m3_to_f(uint8_t b) {
    __nv_fp8_e4m3 x; x.__x = b; return float(x);
}

int main() {
    srand(1);
    std::vector<uint8_t> A(128 * 128), B(16 * 128);
    for (auto& a : A) { __nv_fp8_e4m3 x(((rand() % 2001) - 1000) / 137.0f); a = x.__x; }
    for (auto& b : B) { __nv_fp8_e4m3 x(((rand() % 2001) - 1000) / 511.0f); b = x.__x; }
    std::vector<float> cin(128), cout_(128);
    for (int i = 0; i < 128; ++i) cin[i] = ldexpf(((rand() % 2001) - 1000) / 1000.0f, (i % 20) - 10);
    uint8_t *dA, *dB; float *dD, *dci, *dco;
    cudaMalloc(&dA, A.size()); cudaMalloc(&dB, B.size()); cudaMalloc(&dD, 128 * 16 * 4);
    cudaMalloc(&dci, 512); cudaMalloc(&dco, 512);
    cudaMemcpy(dA, A.data(), A.size(), cudaMemcpyHostToDevice);
    cudaMemcpy(dB, B.data(), B.size(), cudaMemcpyHostToDevice);
    cudaMemcpy(dci, cin.data(), 512, cudaMemcpyHostToDevice);
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    probe<<<1, 128, 64 * 1024>>>(dA, dB, dD, dco, dci);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("CUDA error %s\n", cudaGetErrorString(e)); return 1; }
    std::vector<float> D(128 * 16);
    cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(cout_.data(), dco, 512, cudaMemcpyDeviceToHost);
    double maxerr = 0;
    for (int m = 0; m < 128; ++m)
        for (int n = 0; n < 16; ++n) {
            double ref = 0;
            for (int k = 0; k < 128; ++k) ref += (double)e4m3_to_f(A[m * 128 + k]) * e4m3_to_f(B[n * 128 + k]);
            maxerr = fmax(maxerr, fabs(ref - D[m * 16 + n]));
        }
    double cerr = 0;
    for (int i = 0; i < 128; ++i) {
        __nv_fp8_e4m3 x(cin[i]);
        cerr = fmax(cerr, fabs(float(x) - cout_[i]));
    }
    printf("f8f6f4 e4m3 MMA max err vs fp64 %.3e (D[0]=%f); device cvt mismatch %.3e\n", maxerr, D[0], cerr);
    return 0;
}
