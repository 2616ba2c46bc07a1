// Host-coder sanitizer harness (sanitizers on the coder pool), built by
// tests/test_host_sanitizers.py with -fsanitize=address,undefined and with -fsanitize=thread.
//   mode "fuzz":    every decoder (rANS32 plain / prepared / slabs, rans64) on thousands of
//                   truncated and bit-flipped streams -- a status code, never a fault
//   mode "threads": 8 threads coding and decoding concurrently with shared prepared tables
// Exit status 0 on success; any sanitizer report makes the process fail.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <random>
#include <thread>
#include <vector>

#include "lic.h"

namespace {

constexpr uint32_t C = 24, H = 12, W = 20, L = 32;
constexpr size_t N = (size_t)C * H * W;

struct Fixture {
    std::vector<float> sig;
    std::vector<uint32_t> cdf;
    lic_rans_tables* tab = nullptr;
    std::vector<uint32_t> cdf64;
    std::vector<int32_t> sizes, offs;
    uint32_t stride = 0;
    std::vector<int8_t> sym;
    std::vector<uint8_t> idx;
};

bool build(Fixture& f, uint32_t seed) {
    f.sig.resize(64);
    for (int i = 0; i < 64; ++i) f.sig[i] = (float)std::exp(std::log(0.11) + i * (std::log(64.0) - std::log(0.11)) / 63);
    f.cdf.resize(64 * (2 * L + 2));
    if (lic_cdf_build(f.sig.data(), 64, L, f.cdf.data())) return false;
    if (lic_rans_prepare(f.cdf.data(), 64, 2 * L + 2, -(int)L, &f.tab)) return false;
    f.stride = 2 * (uint32_t)std::ceil(64.0 * 6.2) + 8;
    f.cdf64.assign(64 * (size_t)f.stride, 0);
    f.sizes.assign(64, 0);
    f.offs.assign(64, 0);
    if (lic_cdf64_gaussian(f.sig.data(), 64, 1e-9, f.cdf64.data(), f.stride, f.sizes.data(), f.offs.data())) return false;
    std::mt19937 rng(seed);
    std::normal_distribution<float> nd;
    f.sym.resize(N);
    f.idx.resize(N);
    for (size_t i = 0; i < N; ++i) {
        f.idx[i] = (uint8_t)(rng() % 64);
        const float v = std::round(nd(rng) * f.sig[f.idx[i]] * 1.5f);
        f.sym[i] = (int8_t)std::max(-32.f, std::min(32.f, v));
    }
    return true;
}

// one round of every coder; returns false on a wrong round trip
bool round_trip(const Fixture& f) {
    const lic_shape sh{C, H, W};
    std::vector<uint8_t> out(4 * N + 1024);
    std::vector<int8_t> dec(N);
    size_t len = 0;
    if (lic_rans_encode(f.sym.data(), f.idx.data(), sh, f.cdf.data(), 64, 2 * L + 2, -(int)L, out.data(), out.size(), &len))
        return false;
    if (lic_rans_decode(out.data(), len, f.idx.data(), sh, f.cdf.data(), 64, 2 * L + 2, -(int)L, dec.data()) ||
        std::memcmp(dec.data(), f.sym.data(), N))
        return false;
    for (uint32_t K : {1u, 4u, 8u}) {
        if (lic_rans_encode_slabs(f.tab, f.sym.data(), f.idx.data(), sh, K, out.data(), out.size(), &len)) return false;
        if (lic_rans_decode_slabs(f.tab, out.data(), len, f.idx.data(), sh, K, dec.data()) ||
            std::memcmp(dec.data(), f.sym.data(), N))
            return false;
    }
    std::vector<int32_t> s32(f.sym.begin(), f.sym.end()), i32(f.idx.begin(), f.idx.end()), d32(N);
    if (lic_rans64_encode(s32.data(), i32.data(), N, f.cdf64.data(), 64, f.stride, f.sizes.data(), f.offs.data(),
                          out.data(), out.size(), &len))
        return false;
    if (lic_rans64_decode(out.data(), len, i32.data(), N, f.cdf64.data(), 64, f.stride, f.sizes.data(), f.offs.data(),
                          d32.data()) ||
        std::memcmp(d32.data(), s32.data(), N * 4))
        return false;
    return true;
}

int fuzz() {
    Fixture f;
    if (!build(f, 1)) return 2;
    const lic_shape sh{C, H, W};
    std::vector<uint8_t> s32(4 * N + 1024), s64(4 * N + 1024);
    size_t l32 = 0, l64 = 0, lsl = 0;
    std::vector<uint8_t> ssl(4 * N + 1024);
    std::vector<int32_t> a(f.sym.begin(), f.sym.end()), ix(f.idx.begin(), f.idx.end()), d64(N);
    if (lic_rans_encode_fast(f.tab, f.sym.data(), f.idx.data(), sh, s32.data(), s32.size(), &l32) ||
        lic_rans_encode_slabs(f.tab, f.sym.data(), f.idx.data(), sh, 8, ssl.data(), ssl.size(), &lsl) ||
        lic_rans64_encode(a.data(), ix.data(), N, f.cdf64.data(), 64, f.stride, f.sizes.data(), f.offs.data(),
                          s64.data(), s64.size(), &l64))
        return 3;
    std::mt19937 rng(7);
    std::vector<int8_t> dec(N);
    for (int it = 0; it < 3000; ++it) {
        // truncated (to a random length) and bit-flipped copies of each stream
        for (int which = 0; which < 3; ++which) {
            const std::vector<uint8_t>& src = which == 0 ? s32 : which == 1 ? ssl : s64;
            const size_t len = which == 0 ? l32 : which == 1 ? lsl : l64;
            std::vector<uint8_t> bad(src.begin(), src.begin() + len);
            if (it & 1) bad.resize(rng() % (len + 1));
            for (int k = 0, nf = 1 + (int)(rng() % 4); k < nf && !bad.empty(); ++k) bad[rng() % bad.size()] ^= (uint8_t)(1u << (rng() % 8));
            const uint8_t* p = bad.empty() ? nullptr : bad.data();
            lic_status st;
            if (which == 0) st = lic_rans_decode_fast(f.tab, p, bad.size(), f.idx.data(), sh, dec.data());
            else if (which == 1) st = lic_rans_decode_slabs(f.tab, p, bad.size(), f.idx.data(), sh, 8, dec.data());
            else st = lic_rans64_decode(p, bad.size(), ix.data(), N, f.cdf64.data(), 64, f.stride, f.sizes.data(),
                                        f.offs.data(), d64.data());
            if (st != LIC_OK && st != LIC_ECORRUPT && st != LIC_EINVAL) return 4;
        }
    }
    lic_rans_tables_free(f.tab);
    return 0;
}

int threads() {
    Fixture f;
    if (!build(f, 3)) return 2;
    std::vector<std::thread> th;
    std::vector<int> ok(8, 0);
    for (int i = 0; i < 8; ++i)
        th.emplace_back([&, i] {
            Fixture g;                               // own symbols, shared prepared tables
            build(g, 100 + i);
            lic_rans_tables_free(g.tab);
            g.tab = f.tab;
            int good = 1;
            for (int r = 0; r < 4; ++r) good &= round_trip(g) ? 1 : 0;
            ok[i] = good;
        });
    for (auto& t : th) t.join();
    lic_rans_tables_free(f.tab);
    for (int v : ok)
        if (!v) return 5;
    return 0;
}

}  // namespace

int main(int argc, char** argv) {
    const char* mode = argc > 1 ? argv[1] : "fuzz";
    const int rc = std::strcmp(mode, "threads") == 0 ? threads() : fuzz();
    std::printf("%s rc=%d\n", mode, rc);
    return rc;
}
