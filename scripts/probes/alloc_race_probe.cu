// Probe for compute-sanitizer racecheck's report on the TMEM-address slot (profiles/r2_sanitizer.txt):
// the smallest kernel with the engine's allocation protocol -- warp 2 of each CTA of a 2-CTA
// cluster runs tcgen05.alloc.cta_group::2 (which writes the TMEM address into the CTA's smem
// slot), fence::before_thread_sync, cluster barrier, fence::after_thread_sync, then every thread
// reads the slot.  Nothing else touches shared memory.  If racecheck reports the same
// "tmem_alloc write vs read" hazard here, the report is the tool's model of the tcgen05.alloc
// write, not a race in the engine; the probe also checks that every thread read the same,
// valid address (column 0, lane 0) and that it can be deallocated.
//   nvcc -gencode arch=compute_100a,code=sm_100a -o alloc_race_probe alloc_race_probe.cu
//   compute-sanitizer --tool racecheck ./alloc_race_probe
#include <cstdio>
#include <cuda_runtime.h>

__global__ void __cluster_dims__(2, 1, 1) probe(unsigned* out) {
    __shared__ __align__(16) unsigned slot[4];
    const int warp = threadIdx.x >> 5;
    if (warp == 2) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;"
                     :: "r"((unsigned)__cvta_generic_to_shared(slot)), "r"(128u) : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    asm volatile("barrier.cluster.arrive.release.aligned; barrier.cluster.wait.acquire.aligned;" ::: "memory");
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const unsigned base = *(volatile unsigned*)slot;
    out[blockIdx.x * blockDim.x + threadIdx.x] = base;
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    asm volatile("barrier.cluster.arrive.release.aligned; barrier.cluster.wait.acquire.aligned;" ::: "memory");
    if (warp == 2) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" :: "r"(base), "r"(128u) : "memory");
    }
}

int main() {
    const int blocks = 8, threads = 256;
    unsigned* d;
    cudaMalloc(&d, blocks * threads * sizeof(unsigned));
    cudaMemset(d, 0xff, blocks * threads * sizeof(unsigned));
    probe<<<blocks, threads>>>(d);
    cudaError_t e = cudaDeviceSynchronize();
    unsigned h[blocks * threads];
    cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int b = 0; b < blocks; ++b)
        for (int t = 0; t < threads; ++t)
            if (h[b * threads + t] != h[b * threads] || (h[b * threads] & 0xffff) != 0) ++bad;
    printf("alloc probe: %s, %d threads disagree or read a non-column-aligned address (base of CTA 0: %#x)\n",
           cudaGetErrorString(e), bad, h[0]);
    return e != cudaSuccess || bad;
}
