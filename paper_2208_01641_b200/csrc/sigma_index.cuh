// sigma_index.cuh -- the per-element scale -> CDF-row index of the hyperprior (SPEC.md:187-189,
// DESIGN.md R10): index = #{j in [0, 62] : table_j < max(sigma, 0.11)} over the sorted fp32 scale
// table.  Shared by the h_s L3 epilogue (EP_SIGMA, table in shared memory) and the test kernel
// behind lic_test_sigma_to_index (table in global memory), so the exactness test covers the
// arithmetic the codec runs.
#pragma once

namespace lic {

// A branch-free lower bound over the sorted table in steps 32 .. 1 (the probed position never
// passes 62) -- compact code: the h_s L3 epilogue runs 1-2 tiles per CTA from a cold instruction
// cache.  (Measured slower: a log2 guess corrected by comparisons with its neighbours, whose
// data-dependent loops cost more than the six dependent probes.)
template <class Load>
__device__ __forceinline__ int sigma_to_index(float sigma, const Load& tab) {
    const float s = fmaxf(sigma, 0.11f);
    int lo = 0;
#pragma unroll
    for (int step = 32; step > 0; step >>= 1)
        lo = (tab(lo + step - 1) < s) ? lo + step : lo;
    return lo;
}

}  // namespace lic
