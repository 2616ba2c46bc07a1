// Probe: a 3-D TMA load of a u8 tensor (box 128 B x 19 rows, negative start coordinates;
// the innermost start coordinate must be a multiple of 16 bytes: c0 = 6 is an illegal instruction)
// into shared memory, with and without a 2-CTA cluster launch.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>
#include "../../paper_2208_01641_b200/csrc/ptx.cuh"
using namespace lic;
typedef CUresult (*EncFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                          const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                          CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
__global__ void k(const __grid_constant__ CUtensorMap m, int c0, int c1, int c2, uint8_t* out) {
    __shared__ __align__(1024) uint8_t buf[2432];
    __shared__ __align__(8) uint64_t bar;
    if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
    __syncthreads();
    if (threadIdx.x == 0) {
        mbar_arrive_expect_tx(&bar, 2432);
        tma_load_3d(buf, &m, &bar, c0, c1, c2);
    }
    mbar_wait(&bar, 0);
    for (int i = threadIdx.x; i < 2432; i += blockDim.x) out[blockIdx.x * 2432 + i] = buf[i];
}
int main() {
    const int W = 320, H = 256, B = 2;
    std::vector<uint8_t> h(3 * W * H * B);
    for (size_t i = 0; i < h.size(); ++i) h[i] = (uint8_t)(i * 7 + 3);
    uint8_t *d, *o;
    cudaMalloc(&d, h.size()); cudaMalloc(&o, 2 * 2432);
    cudaMemcpy(d, h.data(), h.size(), cudaMemcpyHostToDevice);
    EncFn enc; cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
    CUtensorMap m;
    cuuint64_t dims[3] = {(cuuint64_t)W * 3, (cuuint64_t)H, (cuuint64_t)B};
    cuuint64_t str[2] = {(cuuint64_t)W * 3, (cuuint64_t)W * 3 * H};
    cuuint32_t box[3] = {128, 19, 1}, es[3] = {1, 1, 1};
    CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode %d\n", (int)r);
    struct Case { int c0, c1, c2, cluster; };
    const Case cases[] = {{0, 5, 0, 0}, {-16, -2, 0, 0}, {944, 250, 1, 0}, {16, -2, 1, 1}, {-16, 5, 1, 1}};
    for (const Case& cs : cases) {
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(2); cfg.blockDim = dim3(128);
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = 2; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
        cfg.attrs = at; cfg.numAttrs = cs.cluster ? 1 : 0;
        cudaLaunchKernelEx(&cfg, k, m, cs.c0, cs.c1, cs.c2, o);
        cudaError_t e = cudaDeviceSynchronize();
        std::vector<uint8_t> ho(2432);
        cudaMemcpy(ho.data(), o, 2432, cudaMemcpyDeviceToHost);
        int bad = 0;
        for (int rr = 0; rr < 19; ++rr) for (int x = 0; x < 128; ++x) {
            int gx = cs.c0 + x, gy = cs.c1 + rr;
            uint8_t ref = (gx >= 0 && gx < 3 * W && gy >= 0 && gy < H) ? h[((size_t)cs.c2 * H + gy) * 3 * W + gx] : 0;
            bad += ho[rr * 128 + x] != ref;
        }
        printf("c (%d, %d, %d) cluster %d: %s bad %d\n", cs.c0, cs.c1, cs.c2, cs.cluster, cudaGetErrorString(e), bad);
        if (e) return 1;
    }
    return 0;
}
