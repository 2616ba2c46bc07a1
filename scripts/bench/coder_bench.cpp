// Host rANS coder micro-benchmark: one C3-sized y plane (192 x 48 x 80) with sigma-indexed rows,
// coded as K channel-slab substreams (lic_rans_encode_slabs / lic_rans_decode_slabs).
//   g++ -O3 -std=c++17 -Iinclude scripts/bench/coder_bench.cpp paper_2208_01641_b200/csrc/host_coder.cpp -o /tmp/cb
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <random>
#include <vector>
#include "lic.h"

int main(int argc, char** argv) {
    const uint32_t C = 192, H = 48, W = 80, L = 32;
    const size_t n = (size_t)C * H * W;
    std::vector<float> sig(64);
    for (int i = 0; i < 64; ++i) sig[i] = (float)std::exp(std::log(0.11) + i * (std::log(256.0) - std::log(0.11)) / 63);
    std::vector<uint32_t> cdf(64 * (2 * L + 2));
    lic_cdf_build(sig.data(), 64, L, cdf.data());
    lic_rans_tables* t = nullptr;
    lic_rans_prepare(cdf.data(), 64, 2 * L + 2, -(int)L, &t);
    std::mt19937 rng(1);
    std::normal_distribution<float> nd;
    std::vector<uint8_t> idx(n);
    std::vector<int8_t> sym(n), dec(n);
    for (size_t i = 0; i < n; ++i) {
        idx[i] = (uint8_t)(rng() % 24);
        float v = std::round(nd(rng) * sig[idx[i]] * 0.6f);
        sym[i] = (int8_t)std::max(-32.f, std::min(32.f, v));
    }
    std::vector<uint8_t> out(2 * n + 1024);
    lic_shape sh{C, H, W};
    for (uint32_t K : {1u, 4u, 8u, 16u, 32u, 64u}) {
        size_t len = 0;
        double be = 1e9, bd = 1e9;
        for (int rep = 0; rep < 15; ++rep) {
            auto t0 = std::chrono::steady_clock::now();
            lic_rans_encode_slabs(t, sym.data(), idx.data(), sh, K, out.data(), out.size(), &len);
            auto t1 = std::chrono::steady_clock::now();
            if (lic_rans_decode_slabs(t, out.data(), len, idx.data(), sh, K, dec.data()) || memcmp(dec.data(), sym.data(), n)) {
                printf("FAIL\n"); return 1;
            }
            auto t2 = std::chrono::steady_clock::now();
            be = std::min(be, std::chrono::duration<double>(t1 - t0).count());
            bd = std::min(bd, std::chrono::duration<double>(t2 - t1).count());
        }
        printf("K=%2u bytes=%zu  enc %.2f ms (%.0f Msym/s)  dec %.2f ms (%.0f Msym/s)\n", K, len, be * 1e3, n / be / 1e6,
               bd * 1e3, n / bd / 1e6);
    }
    return 0;
}
