// conv_umma.cu -- the codec's one GEMM engine: persistent, warp-specialised implicit-GEMM
// convolution / transposed convolution on sm_100a tensor cores (tcgen05 + TMEM + TMA)
// with the layer's nonlinearity fused into the epilogue.
//
// What it computes (Fig. 1 transforms; layer list SPEC.md:319):
//   conv   : out[co][oy][ox] = b[co] + sum W[co][ci][ky][kx] in[ci][s*oy+ky-p][s*ox+kx-p]
//   deconv : stride-2 transposed conv (output_padding 1) as 4 sub-pixel phase GEMMs
//            out[co][2qy+py][2qx+px] = b[co] + sum_{taps of phase} W[..][ky][kx] in[ci][qy+dy][qx+dx]
// then one of the EpKind epilogues: GDN / IGDN as a second tcgen05 MMA of the
// squared activations against gamma followed by rsqrt / sqrt in fp32; quantise;
// sigma -> index; clamp + crop.
//
// Data layout: activations NHWC fp16 as two planes hi = fp16(x), lo = fp16(x - hi)
// (R16); weights W[tap][co][ci] fp16 (exact).  Each pipeline stage carries one
// (tap, 64-channel chunk): A_hi, A_lo (128 px x 64 ch from a strided 5-D TMA box: the
// stride-2 gather and the zero padding are done by the TMA unit) and B (BN x 64).  Two
// MMAs per 16-wide K step (hi, lo) accumulate into one fp32 TMEM accumulator.
//
// Warp roles (640 threads): w0 TMA producer, w1 MMA issuer, w2 TMEM allocator, w3 idle,
// w4-19 epilogue: warp w reads TMEM lanes 32*(w%4).. (= 32 of the tile's 128 pixels) and
// group (w-4)/4 owns one quarter of the output channels.
//
// GDN epilogue: each thread keeps x = acc + b for its half of the channels in registers,
// writes x^2 as fp16 hi/lo back into its own accumulator columns (tcgen05.st), and one
// thread issues norm = x^2 . gamma^T with the A operand read from TMEM (TS MMA) into the
// buffer's norm columns; then y = x * rsqrt(beta + norm) (GDN) or x * sqrt(..) (IGDN).
#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <type_traits>

#include "layer.h"
#include "ptx.cuh"
#include "sigma_index.cuh"

namespace lic {

constexpr int kEpiWarps = 16;                 // 4 per TMEM lane quadrant
constexpr int kEpiGroups = kEpiWarps / 4;     // channel groups (quarters of the N tile)
constexpr int kThreads = 128 + 32 * kEpiWarps;

struct TileCoord { int b, ph, gy0, gx0, nt, split; };

// Tile order: sub-pixel phase fastest, then N tile, x, y, frame -- the 4 phase tiles (and
// the N tiles) of one location run on neighbouring CTAs and share their input via L2.
// The phase is rotated by the location index: with a persistent grid whose size is a multiple
// of 4, CTA c would otherwise always get phase c % 4 (9, 6, 6 or 4 taps) and the kernel
// would run at the speed of its phase-0 CTAs.
// CTA pairs (p.cg = 2) take two horizontally adjacent tiles: rank r gets tile 2*txp + r.
__device__ __forceinline__ int fdiv(int n, uint32_t m, int s) {
    return (int)((__umulhi((uint32_t)n, m) + (uint32_t)n) >> s);
}
// SPLITK: the instantiation may run split-K layers (non-GDN only; run_layer never splits others)
template <bool SPLITK = false>
__device__ __forceinline__ TileCoord decode_tile(const ConvParams& p, int t, int rank) {
    TileCoord c;
    c.split = 0;
    if (SPLITK && p.ksplit > 1) { c.split = t % p.ksplit; t /= p.ksplit; }
    c.ph = t & (p.nphase - 1);  t >>= p.nph_log2;
    if (p.nphase == 4) c.ph = (c.ph + t) & 3;
    int q = fdiv(t, p.fd_nt_m, p.fd_nt_s);
    c.nt = t - q * p.n_ntiles;  t = q;
    q = fdiv(t, p.fd_txs_m, p.fd_txs_s);
    const int tx = (t - q * p.txs) * p.cg + rank;  t = q;
    q = fdiv(t, p.fd_ty_m, p.fd_ty_s);
    const int ty = t - q * p.tiles_y;
    c.b = q;
    c.gx0 = tx * p.tsx;
    c.gy0 = ty * p.tsy;
    return c;
}

// split-K: this tile's slice of the flattened (chunk, parity group, tap) sequence, and one
// group's local tap range [lo, hi) within it (empty: the group is skipped by every role)
struct KRange { int u0, u1, T; };
__device__ __forceinline__ KRange k_range(const ConvParams& p, const TileCoord& tc) {
    KRange k;
    k.T = p.sub4 ? (p.ntaps[0] + p.ntaps[1] + p.ntaps[2] + p.ntaps[3]) : p.ntaps[tc.ph];
    const int U = p.kchunks * k.T;
    k.u0 = p.ksplit > 1 ? tc.split * U / p.ksplit : 0;
    k.u1 = p.ksplit > 1 ? (tc.split + 1) * U / p.ksplit : U;
    return k;
}
__device__ __forceinline__ void group_range(const ConvParams& p, const KRange& k, int c, int gi, int nt, int& lo,
                                            int& hi) {
    const int ub = c * k.T + (p.sub4 ? p.tap0[gi] : 0);
    lo = max(0, k.u0 - ub);
    hi = min(nt, k.u1 - ub);
}

__device__ __forceinline__ uint32_t h2_bits(float a, float b) {
    __half2 h = __floats2half2_rn(a, b);
    return *reinterpret_cast<uint32_t*>(&h);
}
// shared-memory vector load (the aligned dynamic-smem base is a generic pointer, so plain
// dereferences compile to generic LD)
__device__ __forceinline__ float4 lds4(const float* ptr) {
    float4 v;
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(smem_u32(ptr)));
    return v;
}
__device__ __forceinline__ float ldsf(uint32_t addr) {
    float v;
    asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(addr));
    return v;
}
__device__ __forceinline__ uint4 ldsu4(uint32_t addr) {
    uint4 v;
    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr));
    return v;
}
__device__ __forceinline__ uint32_t ldsu(uint32_t addr) {
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr));
    return v;
}
__device__ __forceinline__ uint2 ldsu2(uint32_t addr) {
    uint2 v;
    asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(addr));
    return v;
}
__device__ __forceinline__ void stsu(uint32_t addr, uint32_t v) {
    asm volatile("st.shared.u32 [%0], %1;" :: "r"(addr), "r"(v) : "memory");
}
__device__ __forceinline__ void stsu2(uint32_t addr, uint32_t a, uint32_t b) {
    asm volatile("st.shared.v2.u32 [%0], {%1, %2};" :: "r"(addr), "r"(a), "r"(b) : "memory");
}
// bytes 2i, 2i+1 of w (i = sel: 0x4140 low pair, 0x4342 high pair) -> f16x2 of the integers
// (0x6400 | u is 1024 + u exactly; subtracting 1024 is exact)
__device__ __forceinline__ uint32_t u8pair_to_h2(uint32_t w, uint32_t sel) {
    uint32_t h = __byte_perm(w, 0x64646464u, sel), r;
    asm("sub.rn.f16x2 %0, %1, %2;" : "=r"(r) : "r"(h), "r"(0x64006400u));
    return r;
}
__device__ __forceinline__ uint32_t ldsb(uint32_t addr) {
    uint32_t v;
    asm volatile("ld.shared.u8 %0, [%1];" : "=r"(v) : "r"(addr));
    return v;
}
// 4-byte global -> shared async copy; src_size 0 zero-fills without reading
__device__ __forceinline__ void cp_async4(uint32_t dst, const void* src, uint32_t src_size) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" :: "r"(dst), "l"(src), "r"(src_size) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void stsh(uint32_t addr, uint32_t v) {
    asm volatile("st.shared.u16 [%0], %1;" :: "r"(addr), "h"((unsigned short)v) : "memory");
}
__device__ __forceinline__ void stsf(uint32_t addr, float v) {
    asm volatile("st.shared.f32 [%0], %1;" :: "r"(addr), "f"(v) : "memory");
}
__device__ __forceinline__ void stsu4(uint32_t addr, uint4 v) {
    asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" :: "r"(addr), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
                 : "memory");
}
// fused g_a L1 geometry: 16 x 8 output tile -> 19 x 35 x 3 input patch
constexpr int kL1Wt = 16, kL1Ht = 8;
constexpr int kL1PH = 2 * kL1Ht + 3, kL1PW = (2 * kL1Wt + 3) * 3;    // patch rows, values per row (105)
constexpr int kL1Pitch = 112;                                        // halves per patch row (>= 6*15 + 16)
constexpr uint32_t kL1PlaneBytes = kL1PH * kL1Pitch * 2;             // one fp16 plane of a patch
constexpr int kL1K = 80;                                             // K = 16*ky + 3*kx + c, 5 rows of 16
constexpr int kL1Builders = 96;                                      // warps 0, 2, 3
constexpr int kL1RawWords = 28;                                      // >= (3 + 105) / 4 words loaded per raw row (cp.async)
constexpr int kL1RawPitch = 128;                                     // bytes per raw row (TMA box: 16-byte aligned start + 105 B)
constexpr uint32_t kL1RawBytes = kL1PH * kL1RawPitch;               // one raw u8 patch (2432 B, a multiple of 128)
static_assert(kL1Wt == 16, "build_l1 decodes r -> (r >> 4, r & 15)");
// row-halo g_a L1 (p.l1_rows): tile 8 x 16 output pixels; the raw patch is a 80 B x 35 row TMA
// box (16-byte aligned start + 19 px x 3 B + the 16th sample of the last element); the row halo
// is 35 x 8 elements of one 128-byte SW128 row each (the first 32 bytes used: 16 fp16 samples)
constexpr int kL1RRows = 35;                                         // 2 * 16 + 3 input rows
constexpr int kL1RBox = 80;                                          // bytes per raw row (box width)
constexpr uint32_t kL1RRawBytes = kL1RRows * kL1RBox;                // 2800 B per raw patch
constexpr uint32_t kL1RRawSlot = 2816;                               // raw slot pitch (multiple of 128)
constexpr uint32_t kL1RHaloBytes = kL1RRows * 8 * 128;               // 35840 B per row halo (35 KB)

// MUFU.RSQ without the denormal-input fix-up (GDN/IGDN: beta + n >= beta > 0, normal)
__device__ __forceinline__ float rcp_ftz(float x) {
    float y;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ float rsqrt_ftz(float x) {
    float y;
    asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ float hround(float v) { return __half2float(__float2half_rn(v)); }
// (a, b) -> packed fp16 hi = rn(a, b) and lo = rn(a - hi, b - hi): one pack per plane; the
// residuals a - hi are mixed-precision adds of the packed halves (add.f32.f16: one FHADD each,
// exact -- the same values as converting hi to f32 and subtracting)
__device__ __forceinline__ void split2(float a, float b, uint32_t& hi, uint32_t& lo) {
    const __half2 h = __floats2half2_rn(a, b);
    hi = *reinterpret_cast<const uint32_t*>(&h);
    float ra, rb;
    asm("{\n\t.reg .f16 l, u;\n\tmov.b32 {l, u}, %2;\n\tneg.f16 l, l;\n\tneg.f16 u, u;\n\t"
        "add.rn.f32.f16 %0, l, %3;\n\tadd.rn.f32.f16 %1, u, %4;\n\t}"
        : "=f"(ra), "=f"(rb) : "r"(hi), "f"(a), "f"(b));
    lo = h2_bits(ra, rb);
}
// hi + lo of one packed (hi, lo) fp16 split value pair, half SEL (0 low, 1 high), in f32
template <int SEL>
__device__ __forceinline__ float join_h(uint32_t hi2, uint32_t lo2) {
    float r;
    if constexpr (SEL == 0)
        asm("{\n\t.reg .f16 a, b, c, d;\n\tmov.b32 {a, b}, %1;\n\tmov.b32 {c, d}, %2;\n\t"
            ".reg .f32 t;\n\tcvt.f32.f16 t, c;\n\tadd.rn.f32.f16 %0, a, t;\n\t}" : "=f"(r) : "r"(hi2), "r"(lo2));
    else
        asm("{\n\t.reg .f16 a, b, c, d;\n\tmov.b32 {a, b}, %1;\n\tmov.b32 {c, d}, %2;\n\t"
            ".reg .f32 t;\n\tcvt.f32.f16 t, d;\n\tadd.rn.f32.f16 %0, b, t;\n\t}" : "=f"(r) : "r"(hi2), "r"(lo2));
    return r;
}

// 8 consecutive channels -> one 16-byte fp16 hi vector (+ one lo vector)
__device__ __forceinline__ void split_store8(__half* hi, __half* lo, const float* v) {
    uint4 h, l;
    split2(v[0], v[1], h.x, l.x); split2(v[2], v[3], h.y, l.y);
    split2(v[4], v[5], h.z, l.z); split2(v[6], v[7], h.w, l.w);
    *reinterpret_cast<uint4*>(hi) = h;
    if (lo) *reinterpret_cast<uint4*>(lo) = l;
}

// Activations are stored as fp16 hi + lo planes, whose range ends at 65504 (the same bound
// as the paper's FP16 engines): a value beyond it would become hi = inf,
// lo = -inf and poison the next layer with NaN.  Such values are stored saturated to
// +-65504 and counted (p.range_count, lic_range_count; R16d).
constexpr float kF16Max = 65504.0f;
__device__ __forceinline__ void guard16(float* v, int& ovf) {
    float m = fabsf(v[0]);
#pragma unroll
    for (int j = 1; j < 16; ++j) m = fmaxf(m, fabsf(v[j]));
    if (m > kF16Max) {
#pragma unroll
        for (int j = 0; j < 16; ++j)
            if (fabsf(v[j]) > kF16Max) { ++ovf; v[j] = copysignf(kF16Max, v[j]); }
    }
}
__device__ __forceinline__ void stsb(uint32_t addr, uint32_t v) {
    asm volatile("st.shared.u8 [%0], %1;" :: "r"(addr), "r"(v) : "memory");
}

__device__ __forceinline__ int round_clamp(float v, int L, int& sat) {
    float r = roundf(v);                 // half away from zero (R4)
    if (r > (float)L) { r = (float)L; ++sat; }
    if (r < (float)-L) { r = (float)-L; ++sat; }
    return (int)r;
}

// test-only timeline: event e of the it-th tile of CTA 0 (kTraceEv slots per tile)
constexpr int kTraceEv = kTraceEvents;
constexpr int kTraceTiles = 256;
enum TraceEv { T_MMA_START = 0, T_MMA_END = 1, T_NORM_ISSUE = 2, T_EPI_START = 3, T_EPI_XSQ = 4,
               T_EPI_NORM = 5, T_EPI_END = 6, T_PROD_START = 7,
               T_B_PATCH = 8, T_B_C0_READY = 9, T_B_C0_DONE = 10, T_B_C1_READY = 11, T_B_C1_DONE = 12,
               T_MMA_K0 = 13, T_MMA_KL = 14, T_PEER_B_DONE = 15, T_B_RAW = 16,
               T_EPI_P2 = 17, T_EPI_ACQ = 18, T_EPI_STAGED = 19,
               T_W_HALO = 20, T_W_B = 21, T_B_RAWISS = 22, T_CTA = 23 };
#define LIC_TRACE(it, ev)                                                                         \
    do {                                                                                          \
        if (p.trace && blockIdx.x == 0 && (it) < kTraceTiles)                                     \
            p.trace[(size_t)(it) * kTraceEv + (ev)] = (unsigned long long)clock64();              \
    } while (0)
// the same event recorded by CTA 1 (the pair's peer) -- clock64 is per SM, so only compare
// durations, not absolute times, with CTA 0's events
#define LIC_TRACE_PEER(it, ev)                                                                    \
    do {                                                                                          \
        if (p.trace && blockIdx.x == 1 && (it) < kTraceTiles)                                     \
            p.trace[(size_t)(it) * kTraceEv + (ev)] = (unsigned long long)clock64();              \
    } while (0)

// GC: GDN/IGDN layers only -- 16-column chunks per epilogue group (BN = 64*GC); 0 otherwise.
// CG: 1 = one CTA per 128-pixel tile; 2 = CTA pair (cluster of 2, tcgen05 cta_group::2, M = 256):
//     each CTA loads its own A (or halo) and half of B / gamma, the leader issues the MMAs and
//     commits to both CTAs' barriers, the peer's epilogue arrives remotely on the leader's.
// L1: the fused g_a L1 variant (frame builders, resident weights) -- a separate instantiation,
// so neither variant carries the other's code or register allocation
template <int GC, int CG, bool L1>
__global__ void __launch_bounds__(kThreads, 1)
conv_umma_kernel(const __grid_constant__ CUtensorMap mapA,
                 const __grid_constant__ CUtensorMap mapB,
                 const __grid_constant__ CUtensorMap mapG,
                 const __grid_constant__ CUtensorMap mapOH,
                 const __grid_constant__ CUtensorMap mapOL,
                 const __grid_constant__ CUtensorMap mapO2,
                 const __grid_constant__ CUtensorMap mapO3,
                 const __grid_constant__ ConvParams p)
{
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + p.off_bar);
    uint64_t* empty_bar = full_bar + p.stages;
    uint64_t* tfull_bar = empty_bar + p.stages;     // [2]
    uint64_t* tempty_bar = tfull_bar + 2;           // [2]
    uint64_t* norm_bar = tempty_bar + 2;
    uint64_t* gamma_bar = norm_bar + 1;
    uint64_t* hfull_bar = gamma_bar + 1;            // [4] halo ring
    uint64_t* hempty_bar = hfull_bar + 4;           // [4]
    uint64_t* xsq_bar = hempty_bar + 4;             // epilogue -> MMA warp: x^2 written to TMEM
    uint64_t* wres_bar = xsq_bar + 1;               // resident weights landed
    // the TMEM base address written by tcgen05.alloc, in a 16-byte granule of its own
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + ((p.off_bar + 8u * 34u + 15u) & ~15u));
    uint32_t* xsq_cnt = tmem_slot + 4;              // epilogue warps that wrote x^2 (cumulative)
    // two-group GDN epilogue (p.g2): per accumulator buffer, x^2 written / norm MMAs complete
    uint64_t* xsq2_bar = reinterpret_cast<uint64_t*>(smem + p.off_bar + 320u);    // [2]
    uint64_t* norm2_bar = xsq2_bar + 2;                                            // [2]
    uint64_t* rawfull_bar = norm2_bar + 2;          // [2] fused L1: raw u8 patch landed (TMA)
    float* s_bias = reinterpret_cast<float*>(smem + p.off_par);   // [cout_pad]
    float* s_beta = s_bias + p.BN * p.n_ntiles;                     // [cout_pad]
    float* s_mu = s_beta + p.BN * p.n_ntiles;                       // [cout_pad]
    float* s_tab = s_mu + p.BN * p.n_ntiles;                        // [64]
    uint32_t* s_tapoff = reinterpret_cast<uint32_t*>(s_tab + 64);   // [kMaxTaps] halo window offsets
    // GDN / IGDN: per-pixel exponent of the norm operand, one byte per (pixel, channel group)
    const uint32_t s_xe = smem_u32(s_tapoff + kMaxTaps);            // [128][4] u8

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    constexpr bool kGdn = GC > 0;
    constexpr bool kL1 = L1;                // == p.fuse_l1 (the host dispatches on it)
    constexpr bool kSplitK = GC == 0 && !L1; // split-K layers are ReLU / z-quantise layers
    // two-group GDN epilogue (BN = 128): epilogue warps 4-11 take the even tiles of this CTA,
    // 12-19 the odd ones, each warp 32 pixels x 64 channels; the groups' norm round trips overlap
    const bool g2 = (GC == 2 || GC == 3) && p.g2;
    const uint32_t epi_arrivals = (g2 ? kEpiWarps / 2 : kEpiWarps) * CG;   // per tile
    const int rank = CG == 2 ? (int)cluster_ctarank() : 0;
    const bool leader = rank == 0;
    const int cid = blockIdx.x / CG, ncl = gridDim.x / CG;     // pair (or CTA) index and count
    // barrier address the TMA / epilogue arrivals target: the leader CTA's copy
    auto lbar = [&](uint64_t* b) -> uint32_t { return CG == 2 ? mapa_shared(smem_u32(b), 0) : smem_u32(b); };

    // test-only: CTA entry and setup-done times of CTA 0 (tile slots 0 / 1 of event T_CTA)
    const long long t_entry = p.trace ? clock64() : 0;
    if (threadIdx.x == 0) {
        // fused L1: the 3 builder warps of each CTA arrive on the leader's full barrier
        const uint32_t full_cnt = kL1 ? 3u * CG : 1u;
        for (int s = 0; s < p.stages; ++s) { mbar_init(&full_bar[s], full_cnt); mbar_init(&empty_bar[s], 1); }
        for (int i = 0; i < 2; ++i) { mbar_init(&tfull_bar[i], 1); mbar_init(&tempty_bar[i], epi_arrivals); }
        for (int i = 0; i < 2; ++i) { mbar_init(&xsq2_bar[i], epi_arrivals); mbar_init(&norm2_bar[i], 1); }
        for (int i = 0; i < 2; ++i) mbar_init(&rawfull_bar[i], 1);
        mbar_init(norm_bar, 1);
        mbar_init(gamma_bar, 1);
        for (int i = 0; i < 4; ++i) { mbar_init(&hfull_bar[i], 1); mbar_init(&hempty_bar[i], 1); }
        mbar_init(xsq_bar, kEpiWarps * CG);
        mbar_init(wres_bar, 1);
        *xsq_cnt = 0;
        fence_mbar_init();
    }
    if (warp == 0 && lane == 0) {
        if (!kL1) tma_prefetch_desc(&mapA);
        tma_prefetch_desc(&mapB);
        if (kGdn) tma_prefetch_desc(&mapG);
    }
    if (warp == 2) {
        if constexpr (CG == 2) tmem_alloc_cg2(tmem_slot, (uint32_t)p.tmem_cols);
        else tmem_alloc(tmem_slot, (uint32_t)p.tmem_cols);
    }
    if (warp >= 4) {
        // (the per-channel epilogue constants are staged by the epilogue warps after the setup
        // barrier: their global-load latency stays off the path to the first TMA loads)
        // halo mode: tap t's window starts at halo row (dy+1)*(Wt+2) + dx+1, i.e. this many
        // 16-byte descriptor units past the halo slot
        for (int i = threadIdx.x - 128; i < kMaxTaps; i += 32 * kEpiWarps)
            s_tapoff[i] = (uint32_t)(((p.tap_dy[i] + 1) * p.halo_w + p.tap_dx[i] + 1) * 8);
    }
    if constexpr (kL1) if (!p.l1_rows) {
        // (row halo: no patch or LUT, and the MMAs read only the 32 bytes written per halo row)
        // zero the A stages (K columns >= 80 are never rewritten) and both patch buffers (the
        // row padding halves 105..111 are never rewritten); u8 -> (hi | lo << 16) of u8 / 255
        // (IEEE division, as the oracle), entry 256 = 0 for samples outside the frame
        for (uint32_t i = threadIdx.x; i < p.stages * p.stage_bytes / 16; i += kThreads)
            stsu4(smem_u32(smem) + 16 * i, make_uint4(0, 0, 0, 0));
        for (uint32_t i = threadIdx.x; i < 4 * kL1PlaneBytes / 16; i += kThreads)
            stsu4(smem_u32(smem + p.off_patch) + 16 * i, make_uint4(0, 0, 0, 0));
        for (uint32_t i = threadIdx.x; i < 2 * kL1RawBytes / 16; i += kThreads)    // (cp.async fills 112 of 128 B per row)
            stsu4(smem_u32(smem + p.off_raw) + 16 * i, make_uint4(0, 0, 0, 0));
        uint32_t* lut = reinterpret_cast<uint32_t*>(smem + p.off_lut);
        for (int u = threadIdx.x; u < 257; u += kThreads) {
            uint32_t h = 0, l = 0;
            if (u < 256) {
                if (p.l1_int) h = (uint32_t)__half_as_ushort(__float2half_rn((float)u));   // exact
                else { const float v = __fdiv_rn((float)u, 255.0f); split2(v, 0.0f, h, l); }
            }
            lut[u] = (h & 0xffffu) | (l << 16);
        }
        fence_proxy_async_smem();
    }
    tc_fence_before();
    if constexpr (CG == 2) cluster_sync_all(); else __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    if (threadIdx.x == 0 && p.trace && blockIdx.x == 0) p.trace[T_CTA] = (unsigned long long)t_entry;
    if (threadIdx.x == 0) LIC_TRACE(1, T_CTA);
    if (p.pdl) griddep_launch();          // the next layer may start its prologue on SMs we free

    const uint32_t a_bytes = kBM * kBK * 2;          // 16 KB per activation plane
    const int bnc = p.BN / CG;                        // B (and gamma) rows held by this CTA
    const uint32_t b_bytes = (uint32_t)bnc * kBK * 2;
    const uint32_t idesc = idesc_f16_f32(kBM * CG, (uint32_t)p.BN);
    // TMA into this CTA's smem, completing bytes on the leader's barrier (CG = 2)
    auto ld3 = [&](void* dst, const CUtensorMap* m, uint64_t* bar, int c0, int c1, int c2) {
        if constexpr (CG == 2) tma_load_3d_cg2(dst, m, lbar(bar), c0, c1, c2);
        else tma_load_3d(dst, m, bar, c0, c1, c2);
    };
    auto ld5 = [&](void* dst, const CUtensorMap* m, uint64_t* bar, int c0, int c1, int c2, int c3, int c4) {
        if constexpr (CG == 2) tma_load_5d_cg2(dst, m, lbar(bar), c0, c1, c2, c3, c4);
        else tma_load_5d(dst, m, bar, c0, c1, c2, c3, c4);
    };
    // the leader expects the bytes of both CTAs; the peer's loads only complete_tx
    auto expect = [&](uint64_t* bar, uint32_t bytes) { if (leader) mbar_arrive_expect_tx(bar, bytes * CG); };
    auto commit = [&](uint64_t* bar) {
        if constexpr (CG == 2) umma_commit_pair(bar); else umma_commit(bar);
    };
    auto mma_ss = [&](uint32_t d, uint64_t a, uint64_t b, uint32_t acc) {
        if constexpr (CG == 2) umma_f16_cg2(d, a, b, idesc, acc); else umma_f16(d, a, b, idesc, acc);
    };
    auto mma_ts = [&](uint32_t d, uint32_t a, uint64_t b, uint32_t acc) {
        if constexpr (CG == 2) umma_f16_ts_cg2(d, a, b, idesc, acc); else umma_f16_ts(d, a, b, idesc, acc);
    };

    // ====================== fused g_a L1: im2col A-tile builders (warps 0, 2, 3) ======================
    // K order of the L1 GEMM: k = 16*ky + 3*kx + c (15 values per kernel row + one slot whose
    // weight is zero; 80 used of 128).  Per tile the 19 x 35 x 3 input patch is written to smem
    // already split (fp16 hi and lo planes, rows of 112 halves, zero outside the frame); a K
    // row segment (ky, 8 values from 8h) of pixel (ty, tx) is then 16 contiguous bytes of patch
    // row 2ty + ky at half 6tx + 8h, copied (4 x LDS.32 per plane) into the SW128 A tile.
    auto build_l1 = [&](int bw) {
        const int bt = bw * 32 + lane;
        const uint32_t lut_s = smem_u32(smem + p.off_lut);
        const uint32_t patch_s = smem_u32(smem + p.off_patch);
        const uint32_t raw_s = smem_u32(smem + p.off_raw);
        // u8 frames with 4-byte aligned rows (W % 4 == 0): the patch bytes arrive by cp.async
        // (4-byte words, zero-filled outside the frame -- the frame edges are word boundaries),
        // one tile ahead of the build; otherwise per-sample loads.
        const bool fast = p.fr_u8 && (p.fr_W & 3) == 0;
        const bool lo_on = p.split == 2 && !p.l1_int;     // the lo planes of patch and A tiles
        const bool int_fast = fast && p.l1_int == 2;            // integer samples, no LUT, shifted copy
        // p.raw_tma: the raw patch is one TMA box (128 B x 19 rows of the u8 frame, mapA) starting at
        // the 16-byte boundary at or below the patch's first byte (a TMA start coordinate must be
        // 16-byte aligned in the innermost dimension: scripts/probes/u8_tma_probe.cu), zero fill
        // outside the frame, completing on rawfull_bar
        const bool raw_tma = fast && p.raw_tma;
        auto raw_issue = [&](int tt, int buf) {
            const TileCoord tn = decode_tile<kSplitK>(p, tt, rank);
            if (raw_tma) {
                if (bw == 0 && lane == 0) {
                    mbar_arrive_expect_tx(&rawfull_bar[buf], kL1RawBytes);
                    tma_load_3d(smem + p.off_raw + (uint32_t)buf * kL1RawBytes, &mapA, &rawfull_bar[buf],
                                (3 * (2 * tn.gx0 - 2 - p.fr_left)) & ~15, 2 * tn.gy0 - 2 - p.fr_top, tn.b);
                }
                return;
            }
            const uint8_t* fr = reinterpret_cast<const uint8_t*>(p.frame);
            const int rowb = 3 * p.fr_W;
            const int iyn = 2 * tn.gy0 - 2 - p.fr_top, ws = (3 * (2 * tn.gx0 - 2 - p.fr_left)) >> 2;   // floor
            const uint32_t rb = raw_s + (uint32_t)buf * kL1RawBytes;
            for (int q = bt; q < kL1PH * kL1RawWords; q += kL1Builders) {
                const int r = q / kL1RawWords, w = q - kL1RawWords * r;
                const int iy = iyn + r, gw = 4 * (ws + w);
                const bool ok = iy >= 0 && iy < p.fr_H && gw >= 0 && gw < rowb;
                const uint8_t* src = ok ? fr + ((size_t)tn.b * p.fr_H + iy) * rowb + gw : fr;
                cp_async4(rb + (uint32_t)(r * kL1RawPitch + 4 * w), src, ok ? 4u : 0u);
            }
            cp_async_commit();
        };
        if (p.pdl) griddep_wait();
        if (fast && cid < p.total_tiles) raw_issue(cid, 0);
        int stage = 0;
        uint32_t phase = 0;
        int it = 0;
        for (int t = cid; t < p.total_tiles; t += ncl, ++it) {
            const TileCoord tc = decode_tile<kSplitK>(p, t, rank);
            const uint32_t pbh = patch_s + (uint32_t)((it & 1) * 2 * kL1PlaneBytes), pbl = pbh + kL1PlaneBytes;
            const int iy0 = 2 * tc.gy0 - 2 - p.fr_top, ix0 = 2 * tc.gx0 - 2 - p.fr_left;
            // ---- patch (double-buffered by tile parity; the named barrier of tile it+1 orders
            // every builder's reads of buffer it&1 before anyone rewrites it at tile it+2).
            // All global loads first (independent, in flight together), then split + stores;
            // a thread owns patch columns e0 = bt and e1 = bt + 96 (< 105 for bt < 9).
            const int e0 = bt, e1 = bt + kL1Builders;
            const bool has1 = e1 < kL1PW;
            if (int_fast) {
                // integer samples (l1_int): u8 -> f16 arithmetically, 8 values per item (3 raw
                // words -> one 16-byte store); the lo plane holds a copy shifted by 4 bytes so
                // that every K-row segment below is two 8-byte-aligned loads
                if (raw_tma) {
                    mbar_wait(&rawfull_bar[it & 1], (uint32_t)(it >> 1) & 1u);
                } else {
                    cp_async_wait_all();
                    named_bar_sync_na(4, kL1Builders);                      // raw[it & 1] complete
                }
                if (bw == 0 && lane == 0) LIC_TRACE(it, T_B_RAW);
                // the patch's first byte: at (3 ix0) mod 4 of the raw row (cp.async, word-aligned
                // start) or (3 ix0) mod 16 (TMA, 16-byte aligned start)
                const uint32_t sh = (uint32_t)(3 * ix0) & (raw_tma ? 15u : 3u);
                const uint32_t rw = raw_s + (uint32_t)(it & 1) * kL1RawBytes + (sh & ~3u);
                const uint32_t sel = 0x3210u + (sh & 3u) * 0x1111u;
                for (int q = bt; q < kL1PH * 14; q += kL1Builders) {
                    const int r = q / 14, m = q - 14 * r;
                    const uint32_t src = rw + (uint32_t)(r * kL1RawPitch + 8 * m);
                    const uint2 w01 = ldsu2(src);
                    const uint32_t w2 = ldsu(src + 8);
                    const uint32_t b0 = __byte_perm(w01.x, w01.y, sel), b1 = __byte_perm(w01.y, w2, sel);
                    const uint32_t h0 = u8pair_to_h2(b0, 0x4140u), h1 = u8pair_to_h2(b0, 0x4342u);
                    const uint32_t h2 = u8pair_to_h2(b1, 0x4140u), h3 = u8pair_to_h2(b1, 0x4342u);
                    const uint32_t d = (uint32_t)(r * (2 * kL1Pitch) + 16 * m);
                    stsu4(pbh + d, make_uint4(h0, h1, h2, h3));
                    stsu(pbl + d + 4, h0);
                    stsu2(pbl + d + 8, h1, h2);
                    if (m < 13) stsu(pbl + d + 16, h3);                    // (values 110, 111: unused)
                }
            } else if (fast) {
                if (raw_tma) {
                    mbar_wait(&rawfull_bar[it & 1], (uint32_t)(it >> 1) & 1u);
                } else {
                    cp_async_wait_all();
                    named_bar_sync_na(4, kL1Builders);                      // raw[it & 1] complete
                }
                if (bw == 0 && lane == 0) LIC_TRACE(it, T_B_RAW);
                const uint32_t rb = raw_s + (uint32_t)(it & 1) * kL1RawBytes + ((uint32_t)(3 * ix0) & (raw_tma ? 15u : 3u));
#pragma unroll 4
                for (int r = 0; r < kL1PH; ++r) {
                    const uint32_t w0 = ldsu(lut_s + 4u * ldsb(rb + r * kL1RawPitch + e0));
                    stsh(pbh + 2u * (r * kL1Pitch + e0), w0);
                    if (lo_on) stsh(pbl + 2u * (r * kL1Pitch + e0), w0 >> 16);
                    if (has1) {
                        const uint32_t w1 = ldsu(lut_s + 4u * ldsb(rb + r * kL1RawPitch + e1));
                        stsh(pbh + 2u * (r * kL1Pitch + e1), w1);
                        if (lo_on) stsh(pbl + 2u * (r * kL1Pitch + e1), w1 >> 16);
                    }
                }
            } else if (p.fr_u8) {
                const uint8_t* fr = reinterpret_cast<const uint8_t*>(p.frame);
                const int rowb = 3 * p.fr_W;
                const int gb0 = 3 * ix0 + e0, gb1 = 3 * ix0 + e1;
                const bool c0 = gb0 >= 0 && gb0 < rowb, c1 = has1 && gb1 >= 0 && gb1 < rowb;
                uint32_t u0[kL1PH], u1[kL1PH];
#pragma unroll
                for (int r = 0; r < kL1PH; ++r) {
                    const int iy = iy0 + r;
                    const bool rok = iy >= 0 && iy < p.fr_H;
                    const uint8_t* row = fr + ((size_t)tc.b * p.fr_H + iy) * rowb;
                    u0[r] = (rok && c0) ? (uint32_t)__ldg(row + gb0) : 256u;     // lut[256] = 0
                    u1[r] = (rok && c1) ? (uint32_t)__ldg(row + gb1) : 256u;
                }
#pragma unroll
                for (int r = 0; r < kL1PH; ++r) {
                    const uint32_t w0 = ldsu(lut_s + 4u * u0[r]);                 // hi | lo << 16
                    stsh(pbh + 2u * (r * kL1Pitch + e0), w0);
                    if (lo_on) stsh(pbl + 2u * (r * kL1Pitch + e0), w0 >> 16);
                    if (has1) {
                        const uint32_t w1 = ldsu(lut_s + 4u * u1[r]);
                        stsh(pbh + 2u * (r * kL1Pitch + e1), w1);
                        if (lo_on) stsh(pbl + 2u * (r * kL1Pitch + e1), w1 >> 16);
                    }
                }
            } else {
                const float* fr = reinterpret_cast<const float*>(p.frame);
                const int px0 = e0 / 3, ch0 = e0 - 3 * px0, px1 = e1 / 3, ch1 = e1 - 3 * px1;
                const bool c0 = ix0 + px0 >= 0 && ix0 + px0 < p.fr_W;
                const bool c1 = has1 && ix0 + px1 >= 0 && ix0 + px1 < p.fr_W;
                float v0[kL1PH], v1[kL1PH];
#pragma unroll
                for (int r = 0; r < kL1PH; ++r) {
                    const int iy = iy0 + r;
                    const bool rok = iy >= 0 && iy < p.fr_H;
                    v0[r] = (rok && c0) ? __ldg(fr + (((size_t)tc.b * 3 + ch0) * p.fr_H + iy) * p.fr_W + ix0 + px0) : 0.0f;
                    v1[r] = (rok && c1) ? __ldg(fr + (((size_t)tc.b * 3 + ch1) * p.fr_H + iy) * p.fr_W + ix0 + px1) : 0.0f;
                }
#pragma unroll
                for (int r = 0; r < kL1PH; ++r) {
                    uint32_t h, l;
                    split2(v0[r], v1[r], h, l);
                    stsh(pbh + 2u * (r * kL1Pitch + e0), h);
                    stsh(pbl + 2u * (r * kL1Pitch + e0), l);
                    if (has1) {
                        stsh(pbh + 2u * (r * kL1Pitch + e1), h >> 16);
                        stsh(pbl + 2u * (r * kL1Pitch + e1), l >> 16);
                    }
                }
            }
            named_bar_sync_na(4, kL1Builders);
            if (bw == 0 && lane == 0) LIC_TRACE(it, T_B_PATCH);
            // next tile's raw bytes (its buffer was last read converting tile it-1, before the
            // raw barrier of this tile)
            if (fast && t + ncl < p.total_tiles) raw_issue(t + ncl, (it + 1) & 1);
            if (bw == 0 && lane == 0) LIC_TRACE(it, T_B_RAWISS);
            // ---- A tiles, one stage per 64-column K chunk
            for (int c = 0; c < p.kchunks; ++c) {
                const int kc = c * 64;
                const int nj = max(0, min(8, (kL1K - kc) / 8));             // 16-byte columns with k < 80
                mbar_wait(&empty_bar[stage], phase ^ 1);
                if (bw == 0 && lane == 0) LIC_TRACE(it, c ? T_B_C1_READY : T_B_C0_READY);
                const uint32_t ah = smem_u32(smem + stage * p.stage_bytes), al = ah + a_bytes;
                if (nj > 0) {
                    const int j = bt % nj;                                   // fixed column (96 % nj == 0)
                    const int ky = (kc + 8 * j) >> 4, h8 = (j & 1) * 16;     // kernel row, byte offset in it
                    const int rstep = kL1Builders / nj;
                    for (int r = bt / nj; r < kBM; r += rstep) {
                        const int ty = r >> 4, tx = r & 15;
                        const uint32_t so = (uint32_t)((2 * ty + ky) * (2 * kL1Pitch) + 12 * tx + h8);
                        const uint32_t o = (uint32_t)(r * 128 + ((j ^ (r & 7)) << 4));
                        if (int_fast) {
                            // odd tx: the segment is 4 mod 8 -- read it from the shifted copy
                            const uint32_t sa = (tx & 1) ? pbl + so + 4 : pbh + so;
                            const uint2 v0 = ldsu2(sa), v1 = ldsu2(sa + 8);
                            stsu4(ah + o, make_uint4(v0.x, v0.y, v1.x, v1.y));
                            continue;
                        }
                        uint4 hv;
                        hv.x = ldsu(pbh + so); hv.y = ldsu(pbh + so + 4); hv.z = ldsu(pbh + so + 8); hv.w = ldsu(pbh + so + 12);
                        stsu4(ah + o, hv);
                        if (lo_on) {
                            uint4 lv;
                            lv.x = ldsu(pbl + so); lv.y = ldsu(pbl + so + 4); lv.z = ldsu(pbl + so + 8); lv.w = ldsu(pbl + so + 12);
                            stsu4(al + o, lv);
                        }
                    }
                }
                fence_proxy_async_smem();                             // generic writes -> tensor core
                __syncwarp();
                if (lane == 0) {
                    if constexpr (CG == 2) mbar_arrive_cluster(lbar(&full_bar[stage]));
                    else mbar_arrive(&full_bar[stage]);
                    if (bw == 0) LIC_TRACE(it, c ? T_B_C1_DONE : T_B_C0_DONE);
                    if (bw == 0 && c) LIC_TRACE_PEER(it, T_PEER_B_DONE);
                }
                if (++stage == p.stages) { stage = 0; phase ^= 1; }
            }
            if (bw == 0 && lane == 0) LIC_TRACE(it, T_PROD_START);     // fused L1: tile built
        }
    };
    // row-halo g_a L1 (p.l1_rows; u8 frames, raw TMA, integer samples -- layer.h): per tile one
    // raw TMA box (prefetched two tiles ahead into 2 slots) -> one row halo in stage `stage`
    auto build_l1_rows = [&](int bw) {
        const int bt = bw * 32 + lane;
        const uint32_t raw_s = smem_u32(smem + p.off_raw);
        auto raw_issue = [&](int tt, int buf) {
            if (bw != 0 || lane != 0 || tt >= p.total_tiles) return;
            const TileCoord tn = decode_tile<kSplitK>(p, tt, rank);
            fence_proxy_async_smem();                 // the builders' reads of this slot precede the TMA write
            mbar_arrive_expect_tx(&rawfull_bar[buf], kL1RRawBytes);
            tma_load_3d(smem + p.off_raw + (uint32_t)buf * kL1RRawSlot, &mapA, &rawfull_bar[buf],
                        (3 * (2 * tn.gx0 - 2 - p.fr_left)) & ~15, 2 * tn.gy0 - 2 - p.fr_top, tn.b);
        };
        if (p.pdl) griddep_wait();
        raw_issue(cid, 0);
        raw_issue(cid + ncl, 1);
        int stage = 0;
        uint32_t phase = 0;
        int it = 0;
        for (int t = cid; t < p.total_tiles; t += ncl, ++it) {
            const TileCoord tc = decode_tile<kSplitK>(p, t, rank);
            const int ix0 = 2 * tc.gx0 - 2 - p.fr_left;
            // the patch's first byte inside the 16-byte aligned box
            const uint32_t sh = (uint32_t)(3 * ix0) & 15u;
            const uint32_t rb = raw_s + (uint32_t)(it & 1) * kL1RRawSlot;
            mbar_wait(&rawfull_bar[it & 1], (uint32_t)(it >> 1) & 1u);
            if (bw == 0 && lane == 0) LIC_TRACE(it, T_B_RAW);
            mbar_wait(&empty_bar[stage], phase ^ 1);
            if (bw == 0 && lane == 0) LIC_TRACE(it, T_B_C0_READY);
            const uint32_t hb = smem_u32(smem + stage * p.stage_bytes);
            for (int e = bt; e < kL1RRows * 8; e += kL1Builders) {
                const int iy = e >> 3, tx = e & 7;
                const uint32_t o = sh + 6u * (uint32_t)tx;                 // byte offset in the raw row
                const uint32_t src = rb + (uint32_t)iy * kL1RBox + (o & ~3u);
                const uint32_t w0 = ldsu(src), w1 = ldsu(src + 4), w2 = ldsu(src + 8), w3 = ldsu(src + 12),
                               w4 = ldsu(src + 16);
                const uint32_t s8 = (o & 3u) * 8u;
                const uint32_t a0 = __funnelshift_r(w0, w1, s8), a1 = __funnelshift_r(w1, w2, s8);
                const uint32_t a2 = __funnelshift_r(w2, w3, s8), a3 = __funnelshift_r(w3, w4, s8);
                // samples 0-7 -> logical 16-byte chunk 0, 8-15 -> chunk 1 (SW128: chunk c of row e at c ^ (e & 7))
                const uint32_t d = hb + (uint32_t)e * 128u;
                stsu4(d + ((uint32_t)tx << 4),
                      make_uint4(u8pair_to_h2(a0, 0x4140u), u8pair_to_h2(a0, 0x4342u),
                                 u8pair_to_h2(a1, 0x4140u), u8pair_to_h2(a1, 0x4342u)));
                stsu4(d + (((uint32_t)tx ^ 1u) << 4),
                      make_uint4(u8pair_to_h2(a2, 0x4140u), u8pair_to_h2(a2, 0x4342u),
                                 u8pair_to_h2(a3, 0x4140u), u8pair_to_h2(a3, 0x4342u)));
            }
            fence_proxy_async_smem();                             // generic writes -> tensor core
            __syncwarp();
            if (lane == 0) {
                if constexpr (CG == 2) mbar_arrive_cluster(lbar(&full_bar[stage]));
                else mbar_arrive(&full_bar[stage]);
                if (bw == 0) LIC_TRACE(it, T_B_C0_DONE);
            }
            if (++stage == p.stages) { stage = 0; phase ^= 1; }
            // every builder has read raw slot it & 1: it takes tile it + 2's patch
            named_bar_sync_na(4, kL1Builders);
            raw_issue(t + 2 * ncl, it & 1);
            if (bw == 0 && lane == 0) LIC_TRACE(it, T_PROD_START);
        }
    };
    auto build_l1_any = [&](int bw) {
        if (p.l1_rows) build_l1_rows(bw); else build_l1(bw);
    };

    if (kL1 && warp == 2) {
        if constexpr (kL1) build_l1_any(1);
    } else if (warp == 0) {
        // ====================== TMA producer (weights; activations unless halo mode) ======================
        // warp-uniform loop; one elected lane issues (keeps coordinates in uniform registers)
        if (kGdn) {
            // gamma (Cout x Cout fp16, K-major rows; BN/64 = GC chunks of 64 columns), resident
            if (elect_one()) {
                expect(gamma_bar, (uint32_t)GC * b_bytes);
                for (int c = 0; c < GC; ++c)         // this CTA's half of gamma's rows (CG = 2)
                    ld3(smem + p.off_gamma + c * b_bytes, &mapG, gamma_bar, c * kBK, rank * bnc, 0);
            }
            __syncwarp();
        }
        if (p.wres) {
            // every (tap, chunk) weight tile, once per CTA: tile (w, c) at (w * kchunks + c) * b_bytes
            if (elect_one()) {
                const int nw = p.ntaps[0];
                expect(wres_bar, (uint32_t)(nw * p.kchunks) * b_bytes);
                for (int w = 0; w < nw; ++w)
                    for (int c = 0; c < p.kchunks; ++c)
                        ld3(smem + p.off_wres + (w * p.kchunks + c) * b_bytes, &mapB, wres_bar, c * kBK, rank * bnc,
                                    p.tap_w[w]);
            }
            __syncwarp();
        }
        // activations below come from the previous kernel; in halo mode this warp streams only
        // weights (constant), so its ring fills while the previous layer is still finishing
        if (p.pdl && !p.halo) griddep_wait();
        int stage = 0;
        uint32_t phase = 0;
        int pit = 0;
        // (resident weights: only the gather mode still streams A tiles from here)
        for (int t = cid; !kL1 && t < p.total_tiles && (!p.wres || p.gather); t += ncl, ++pit) {
            TileCoord tc = decode_tile<kSplitK>(p, t, rank);
            const int nt = p.ntaps[tc.ph], t0 = p.tap0[tc.ph];
            if (lane == 0) LIC_TRACE(pit, T_PROD_START);
            if (p.halo) {
                // chunk-outer, tap-inner weight tiles (halos come from warp 3); p.tps consecutive
                // taps share a stage (one barrier wait per 8 * tps MMAs)
                // (sub4: the 4 parity groups of each chunk in turn)
                const KRange kr = k_range(p, tc);
                for (int c = 0; c < p.kchunks; ++c)
                    for (int gi = 0; gi < (p.sub4 ? 4 : 1); ++gi) {
                        const int gnt = p.sub4 ? p.ntaps[gi] : nt, gt0 = p.sub4 ? p.tap0[gi] : t0;
                        int tlo, thi;
                        group_range(p, kr, c, gi, gnt, tlo, thi);
                        for (int ti = tlo; ti < thi; ti += p.tps) {
                            const int ntp = min(p.tps, thi - ti);
                            mbar_wait(&empty_bar[stage], phase ^ 1);
                            if (elect_one()) {
                                expect(&full_bar[stage], b_bytes * (uint32_t)ntp);
                                for (int u = 0; u < ntp; ++u)
                                    ld3(smem + stage * p.stage_bytes + u * b_bytes, &mapB, &full_bar[stage], c * kBK,
                                        tc.nt * p.BN + rank * bnc, p.tap_w[gt0 + ti + u]);
                            }
                            __syncwarp();
                            if (++stage == p.stages) { stage = 0; phase ^= 1; }
                        }
                    }
                continue;
            }
            for (int ti = 0; ti < nt; ++ti) {
                const int x0 = p.stride * tc.gx0 + p.tap_dx[t0 + ti];
                const int y0 = p.stride * tc.gy0 + p.tap_dy[t0 + ti];
                const int wt = p.tap_w[t0 + ti];
                for (int c = 0; c < p.kchunks; ++c) {
                    mbar_wait(&empty_bar[stage], phase ^ 1);
                    uint8_t* st = smem + stage * p.stage_bytes;
                    if (elect_one()) {
                        expect(&full_bar[stage], a_bytes * p.split + (p.wres ? 0u : b_bytes));
                        ld5(st, &mapA, &full_bar[stage], c * kBK, x0, y0, tc.b, 0);
                        if (p.split == 2) ld5(st + a_bytes, &mapA, &full_bar[stage], c * kBK, x0, y0, tc.b, 1);
                        if (!p.wres)
                            ld3(st + a_bytes * p.split, &mapB, &full_bar[stage], c * kBK, tc.nt * p.BN + rank * bnc, wt);
                    }
                    __syncwarp();
                    if (++stage == p.stages) { stage = 0; phase ^= 1; }
                }
            }
        }
        if constexpr (kL1) build_l1_any(0);
    } else if (warp == 3) {
        // ====================== halo producer (halo mode) ======================
        if constexpr (kL1) build_l1_any(2);
        if (!kL1 && p.halo) {
            if (p.pdl) griddep_wait();
            int hs = 0;
            uint32_t hphase = 0;
            const bool hlo = p.split == 2 && !p.a_hi_only;      // load the lo plane
            const uint32_t hbytes = (uint32_t)p.halo_w * (p.Ht + 2) * 128 * (hlo ? 2 : 1);
            for (int t = cid; t < p.total_tiles; t += ncl) {
                TileCoord tc = decode_tile<kSplitK>(p, t, rank);
                const KRange kr = k_range(p, tc);
                for (int c = 0; c < p.kchunks; ++c)
                  for (int gi = 0; gi < (p.sub4 ? 4 : 1); ++gi) {
                    {
                        int tlo, thi;
                        group_range(p, kr, c, gi, p.sub4 ? p.ntaps[gi] : p.ntaps[tc.ph], tlo, thi);
                        if (tlo >= thi) continue;                       // no tap of this K slice
                    }
                    // sub4: parity sub-grid (py, px) = (gi >> 1, gi & 1), rows / columns gy0 - 1 ..
                    // of the sub-grid = input 2 * (gy0 - 1) + py .. in steps of 2 (the map's stride)
                    const int hx = p.sub4 ? 2 * (tc.gx0 - 1) + (gi & 1) : tc.gx0 - 1;
                    const int hy = p.sub4 ? 2 * (tc.gy0 - 1) + (gi >> 1) : tc.gy0 - 1;
                    mbar_wait(&hempty_bar[hs], hphase ^ 1);
                    uint8_t* hb = smem + p.off_halo + hs * (p.halo_planes * p.halo_plane_bytes);
                    if (elect_one()) {
                        expect(&hfull_bar[hs], hbytes);
                        ld5(hb, &mapA, &hfull_bar[hs], c * kBK, hx, hy, tc.b, 0);
                        if (hlo) ld5(hb + p.halo_plane_bytes, &mapA, &hfull_bar[hs], c * kBK, hx, hy, tc.b, 1);
                    }
                    __syncwarp();
                    if (++hs == p.halo_slots) { hs = 0; hphase ^= 1; }
                  }
            }
        }
    } else if (warp == 1) {
        // ====================== MMA issuer ======================
        // Warp-uniform; one elected lane issues each batch of tcgen05.mma.
        // GDN/IGDN: the norm MMAs (x^2 . gamma^T, A from TMEM) of tile i are issued HERE, as soon
        // as the epilogue has written x^2 (xsq_bar), between K-steps of tile i+1 -- the tensor
        // pipe runs MMAs in issue order, so issuing them from the epilogue would queue them
        // behind the whole next main loop.
        int stage = 0;
        uint32_t phase = 0;
        int hs = 0;
        uint32_t hphase = 0;
        int it = 0;
        int pend = 0;                       // a tile's norm MMAs are outstanding
        uint32_t pend_dcol = 0, xsq_phase = 0;
        int pend_it = 0;
        bool gamma_ready = false;
        auto issue_norm = [&](uint64_t* done_bar) {
            if (!gamma_ready) { mbar_wait(gamma_bar, 0); gamma_ready = true; }
            tc_fence_after();
            constexpr int G = 16 * (GC > 0 ? GC : 1);
            const uint32_t ncol = tmem_base + pend_dcol + (uint32_t)p.BN;
            const uint32_t gbase = smem_u32(smem + p.off_gamma);
            if (elect_one()) {
#pragma unroll
                for (int kk = 0; kk < 4 * GC; ++kk) {           // K = BN in steps of 16
                    const int k0 = 16 * kk, gg = k0 / G, o = k0 - gg * G;
                    const uint32_t ahi = tmem_base + pend_dcol + gg * G + o / 2;
                    const uint32_t alo = ahi + G / 2;
                    const uint64_t bd = sdesc_sw128(gbase + (k0 / 64) * b_bytes) + 2 * (kk & 3);
                    mma_ts(ncol, ahi, bd, kk != 0);
                    mma_ts(ncol, alo, bd, 1u);
                }
                commit(done_bar);
            }
            __syncwarp();
            if (lane == 0) LIC_TRACE(pend_it, T_NORM_ISSUE);
            pend = 0;
        };
        int xsq_seen = 0;              // tiles whose x^2 the MMA warp has consumed
        // two-group epilogue: tiles whose main MMAs are committed / whose norm MMAs are issued
        // (in tile order; tile n uses accumulator buffer n & 1, the (n >> 1)-th phase of its barriers)
        int g2_committed = 0;
        (void)g2_committed;
        auto poll_norm = [&]() {       // cheap volatile smem read; the mbarrier wait then completes at once
            if (g2) return;                                  // the epilogue issues its own norm MMAs
            if (kGdn && pend && *reinterpret_cast<volatile uint32_t*>(xsq_cnt) >= (uint32_t)(kEpiWarps * CG * (xsq_seen + 1))) {
                mbar_wait(xsq_bar, xsq_phase);
                xsq_phase ^= 1;
                ++xsq_seen;
                issue_norm(norm_bar);
            }
        };
        // blocking waits of the MMA warp keep polling for a pending norm (GDN), so that the
        // norm of tile i is not held back while the warp waits for tile i+1's operands
        auto wait_poll = [&](uint64_t* bar, uint32_t par) {
            if constexpr (kGdn) {
                if (g2 && !p.mma_spin) { mbar_wait(bar, par); return; }   // norms issued by the epilogue (g2)
                if (mbar_test(bar, par)) return;
                const long long t0 = clock64();
                while (!mbar_test(bar, par)) {
                    if (!g2) poll_norm();
                    if (clock64() - t0 > (1ll << 35)) __trap();      // protocol bug: fail loudly
                }
            } else {
                mbar_wait(bar, par);
            }
        };
        if (p.wres && leader) mbar_wait(wres_bar, 0);      // the peer's bytes land on the leader's barrier
        for (int t = cid; t < p.total_tiles && leader; t += ncl, ++it) {
            TileCoord tc = decode_tile<kSplitK>(p, t, rank);
            const int buf = (p.n_accbuf == 2) ? (it & 1) : 0;
            const uint32_t use = (p.n_accbuf == 2) ? (uint32_t)(it >> 1) : (uint32_t)it;
            if (kGdn && !g2 && pend && p.n_accbuf == 1) { mbar_wait(xsq_bar, xsq_phase); xsq_phase ^= 1; ++xsq_seen; issue_norm(norm_bar); }
            wait_poll(&tempty_bar[buf], (use & 1) ^ 1);
            tc_fence_after();
            if (lane == 0) LIC_TRACE(it, T_MMA_START);
            const uint32_t d = tmem_base + (uint32_t)(buf * p.acc_stride);
            long long w_halo = 0, w_b = 0;          // trace only: cycles waiting for operands
            // halo mode, streamed weights, 2 or 3 taps per stage, no trace: the lean issue loop --
            // tap window offsets from the kernel parameters (uniform registers), the stage count
            // compile-time, no per-stage parameter tests
            auto halo_fast = [&](auto tps_c, auto lo_c, auto split_c) {
                constexpr int TPS = decltype(tps_c)::value;
                constexpr bool LO = decltype(lo_c)::value;
                constexpr bool SPLIT = decltype(split_c)::value;   // a K slice (split-K layers)
                const uint32_t sbo = (uint32_t)p.halo_w * 128;
                const uint32_t hstride = (uint32_t)p.halo_planes * p.halo_plane_bytes;
                const uint64_t lo16 = p.halo_plane_bytes >> 4;
                const uint64_t bstep16 = b_bytes >> 4;
                const uint32_t halo0 = smem_u32(smem + p.off_halo), stage0 = smem_u32(smem);
                const int ngr = p.sub4 ? 4 : 1;
                KRange kr;
                if constexpr (SPLIT) kr = k_range(p, tc);
                bool first = true;                         // the K slice's first MMA overwrites the accumulator
                for (int c = 0; c < p.kchunks; ++c)
                    for (int gi = 0; gi < ngr; ++gi) {
                        const int nt = p.sub4 ? p.ntaps[gi] : p.ntaps[tc.ph], t0 = p.sub4 ? p.tap0[gi] : p.tap0[tc.ph];
                        int tlo = 0, thi = nt;
                        if constexpr (SPLIT) {
                            group_range(p, kr, c, gi, nt, tlo, thi);
                            if (tlo >= thi) continue;
                        }
                        long long tw0 = p.trace ? clock64() : 0;
                        wait_poll(&hfull_bar[hs], hphase);
                        if (p.trace) w_halo += clock64() - tw0;
                        tc_fence_after();
                        if (lane == 0 && c == 0 && gi == 0) LIC_TRACE(it, T_MMA_K0);
                        const uint64_t ahb = sdesc_sw128_sbo(halo0 + (uint32_t)hs * hstride, sbo);
                        for (int ti = tlo; ti < thi; ti += TPS) {
                            const int ntp = min(TPS, thi - ti);
                            long long tw1 = p.trace ? clock64() : 0;
                            wait_poll(&full_bar[stage], phase);
                            if (p.trace) w_b += clock64() - tw1;
                            tc_fence_after();
                            const uint64_t bdb = sdesc_sw128(stage0 + (uint32_t)stage * p.stage_bytes);
                            if (elect_one()) {
                                const uint32_t acc0 = SPLIT ? (first ? 0u : 1u) : ((c | gi | ti) != 0);
#pragma unroll
                                for (int u = 0; u < TPS; ++u) {
                                    if (u < ntp) {
                                        const uint64_t ah = ahb + p.tapoff[t0 + ti + u];
                                        const uint64_t bd = bdb + (uint64_t)u * bstep16;
#pragma unroll
                                        for (int kk = 0; kk < kBK / 16; ++kk) {
                                            mma_ss(d, ah + 2 * kk, bd + 2 * kk, (u | kk) ? 1u : acc0);
                                            if constexpr (LO) mma_ss(d, ah + lo16 + 2 * kk, bd + 2 * kk, 1u);
                                        }
                                    }
                                }
                                commit(&empty_bar[stage]);
                            }
                            __syncwarp();
                            if constexpr (SPLIT) first = false;
                            if (++stage == p.stages) { stage = 0; phase ^= 1; }
                            poll_norm();
                        }
                        if (elect_one()) commit(&hempty_bar[hs]);
                        __syncwarp();
                        if (++hs == p.halo_slots) { hs = 0; hphase ^= 1; }
                    }
            };
            const bool fast_halo = !kL1 && p.halo && !p.wres && (p.tps == 2 || p.tps == 3);
            if constexpr (kL1) {
                // (fused L1: the plain K loop below)
            }
            if (fast_halo) {
                using I2 = std::integral_constant<int, 2>;
                using I3 = std::integral_constant<int, 3>;
                using BT = std::integral_constant<bool, true>;
                using BF = std::integral_constant<bool, false>;
                const bool lo_mma = p.split == 2 && !p.a_hi_only;
                if (kSplitK && p.ksplit > 1) {
                    if (p.tps == 2) { if (lo_mma) halo_fast(I2{}, BT{}, BT{}); else halo_fast(I2{}, BF{}, BT{}); }
                    else { if (lo_mma) halo_fast(I3{}, BT{}, BT{}); else halo_fast(I3{}, BF{}, BT{}); }
                } else {
                    if (p.tps == 2) { if (lo_mma) halo_fast(I2{}, BT{}, BF{}); else halo_fast(I2{}, BF{}, BF{}); }
                    else { if (lo_mma) halo_fast(I3{}, BT{}, BF{}); else halo_fast(I3{}, BF{}, BF{}); }
                }
            } else if (!kL1 && p.halo) {
                const uint32_t sbo = (uint32_t)p.halo_w * 128;
                const bool lo_mma = p.split == 2 && !p.a_hi_only;
                for (int c = 0; c < p.kchunks; ++c)
                  for (int gi = 0; gi < (p.sub4 ? 4 : 1); ++gi) {
                    const int nt = p.sub4 ? p.ntaps[gi] : p.ntaps[tc.ph], t0 = p.sub4 ? p.tap0[gi] : p.tap0[tc.ph];
                    long long tw0 = p.trace ? clock64() : 0;
                    wait_poll(&hfull_bar[hs], hphase);
                    if (p.trace) w_halo += clock64() - tw0;
                    tc_fence_after();
                    if (lane == 0 && c == 0 && gi == 0) LIC_TRACE(it, T_MMA_K0);
                    const uint32_t hb = smem_u32(smem + p.off_halo + hs * (p.halo_planes * p.halo_plane_bytes));
                    // descriptors of the halo slot (hi, lo planes); a tap's window adds its row
                    // offset (s_tapoff: 16-byte units, no carry out of the 14-bit address field)
                    const uint64_t ahb = sdesc_sw128_sbo(hb, sbo);
                    const uint64_t alb = ahb + (p.halo_plane_bytes >> 4);
                    // p.tps taps per weight stage: one barrier wait / fence / commit per 8 * tps MMAs
                    // (the issue loop, not the tensor pipe, is what waits between groups)
                    const int tps = p.wres ? 1 : p.tps;
                    for (int ti = 0; ti < nt; ti += tps) {
                        const int ntp = min(tps, nt - ti);
                        uint32_t bsm;
                        if (p.wres) {
                            bsm = smem_u32(smem + p.off_wres + ((t0 + ti) * p.kchunks + c) * b_bytes);
                        } else {
                            long long tw1 = p.trace ? clock64() : 0;
                            wait_poll(&full_bar[stage], phase);
                            if (p.trace) w_b += clock64() - tw1;
                            tc_fence_after();
                            bsm = smem_u32(smem + stage * p.stage_bytes);
                        }
                        const uint64_t bdb = sdesc_sw128(bsm);
                        uint32_t toff[kMaxTps];
#pragma unroll
                        for (int u = 0; u < kMaxTps; ++u) toff[u] = u < ntp ? s_tapoff[t0 + ti + u] : 0u;
                        if (elect_one()) {
                            const uint32_t acc0 = (c | gi | ti) != 0;
                            // two copies of the issue loop (hi + lo planes / hi only): no predicated
                            // MMAs, so the descriptors stay in uniform registers
                            if (lo_mma) {
#pragma unroll
                                for (int u = 0; u < kMaxTps; ++u) {
                                    if (u < ntp) {
                                        const uint64_t ah = ahb + toff[u], al = alb + toff[u];
                                        const uint64_t bd = bdb + (uint64_t)(u * (b_bytes >> 4));
#pragma unroll
                                        for (int kk = 0; kk < kBK / 16; ++kk) {
                                            mma_ss(d, ah + 2 * kk, bd + 2 * kk, (u | kk) ? 1u : acc0);
                                            mma_ss(d, al + 2 * kk, bd + 2 * kk, 1u);
                                        }
                                    }
                                }
                            } else {
#pragma unroll
                                for (int u = 0; u < kMaxTps; ++u) {
                                    if (u < ntp) {
                                        const uint64_t ah = ahb + toff[u];
                                        const uint64_t bd = bdb + (uint64_t)(u * (b_bytes >> 4));
#pragma unroll
                                        for (int kk = 0; kk < kBK / 16; ++kk)
                                            mma_ss(d, ah + 2 * kk, bd + 2 * kk, (u | kk) ? 1u : acc0);
                                    }
                                }
                            }
                            if (!p.wres) commit(&empty_bar[stage]);
                        }
                        __syncwarp();
                        if (!p.wres && ++stage == p.stages) { stage = 0; phase ^= 1; }
                        poll_norm();
                    }
                    if (elect_one()) commit(&hempty_bar[hs]);
                    __syncwarp();
                    if (++hs == p.halo_slots) { hs = 0; hphase ^= 1; }
                }
            } else if (kL1 && p.l1_rows) {
                // row-halo g_a L1: kernel row ky is one K = 16 MMA -- A = the halo rows 2 ty + ky
                // (window start ky * 8 rows, 8-row groups every 2 halo row-blocks), B = K columns
                // 16 ky .. 16 ky + 15 of the resident weights (chunk ky / 4, step ky % 4)
                wait_poll(&full_bar[stage], phase);
                tc_fence_after();
                if (lane == 0) LIC_TRACE(it, T_MMA_K0);
                const uint32_t st = smem_u32(smem + stage * p.stage_bytes);
                const uint32_t wb = smem_u32(smem + p.off_wres);
                if (elect_one()) {
#pragma unroll
                    for (int ky = 0; ky < 5; ++ky)
                        mma_ss(d, sdesc_sw128_sbo(st + (uint32_t)ky * 1024u, 2048u),
                               sdesc_sw128(wb + (uint32_t)(ky >> 2) * b_bytes) + 2 * (ky & 3), ky != 0);
                    commit(&empty_bar[stage]);
                }
                __syncwarp();
                if (++stage == p.stages) { stage = 0; phase ^= 1; }
                poll_norm();
            } else {
                const int nk = p.ntaps[tc.ph] * p.kchunks;
                const int t0k = p.tap0[tc.ph] * p.kchunks;            // resident weights: tile (tap, chunk)
                for (int k = 0; k < nk; ++k) {
                    wait_poll(&full_bar[stage], phase);
                    tc_fence_after();
                    if (lane == 0 && k == 0) LIC_TRACE(it, T_MMA_K0);
                    if (lane == 0 && k == nk - 1) LIC_TRACE(it, T_MMA_KL);
                    const uint32_t st = smem_u32(smem + stage * p.stage_bytes);
                    const uint64_t ah = sdesc_sw128(st);
                    const uint64_t al = sdesc_sw128(st + a_bytes);
                    const uint64_t bd = p.wres ? sdesc_sw128(smem_u32(smem + p.off_wres + (t0k + k) * b_bytes))
                                               : sdesc_sw128(st + a_bytes * p.split);
                    if (elect_one()) {
#pragma unroll
                        for (int kk = 0; kk < kBK / 16; ++kk) {
                            // +32 bytes per 16-element K step inside the 128-byte swizzle row
                            mma_ss(d, ah + 2 * kk, bd + 2 * kk, (k | kk) != 0);
                            if (p.split == 2 && !p.l1_int) mma_ss(d, al + 2 * kk, bd + 2 * kk, 1u);
                        }
                        commit(&empty_bar[stage]);
                    }
                    __syncwarp();
                    if (++stage == p.stages) { stage = 0; phase ^= 1; }
                    poll_norm();
                }
            }
            if (elect_one()) commit(&tfull_bar[buf]);
            __syncwarp();
            if (lane == 0) LIC_TRACE(it, T_MMA_END);
            if (lane == 0 && p.trace && blockIdx.x == 0 && it < kTraceTiles) {
                p.trace[(size_t)it * kTraceEv + T_W_HALO] = (unsigned long long)w_halo;
                p.trace[(size_t)it * kTraceEv + T_W_B] = (unsigned long long)w_b;
            }

            if (g2) {
                g2_committed = it + 1;
            } else if (kGdn) {
                // the previous tile's norm must be issued before this one becomes pending
                if (pend) { mbar_wait(xsq_bar, xsq_phase); xsq_phase ^= 1; ++xsq_seen; issue_norm(norm_bar); }
                pend = 1;
                pend_it = it;
                pend_dcol = (uint32_t)(buf * p.acc_stride);
            }
        }
        if (kGdn && !g2 && pend && leader) { mbar_wait(xsq_bar, xsq_phase); xsq_phase ^= 1; ++xsq_seen; issue_norm(norm_bar); }
    } else if (warp >= 4) {
        // ====================== epilogue ======================
        {
            // per-channel epilogue constants, staged once per CTA (visible to every epilogue warp
            // after the named barrier; nobody else reads them)
            const int np = p.BN * p.n_ntiles;
            for (int i = threadIdx.x - 128; i < np; i += 32 * kEpiWarps) {
                const bool in = i < p.Cout;
                s_bias[i] = in ? p.bias[i] : 0.0f;
                s_beta[i] = (in && p.beta) ? p.beta[i] : 0.0f;
                s_mu[i] = (in && p.mu) ? p.mu[i] : 0.0f;
            }
            for (int i = threadIdx.x - 128; i < 64; i += 32 * kEpiWarps) s_tab[i] = p.table ? p.table[i] : 0.0f;
            named_bar_sync(15, 32 * kEpiWarps);
        }
        if (p.pdl) griddep_wait();                  // global writes only after the previous kernel
        const int q = warp & 3;                     // TMEM lane quadrant
        const int g = (warp - 4) >> 2;              // channel group (quarter)
        const int r = q * 32 + lane;                // tile row (pixel) of this thread
        const uint32_t lane_off = (uint32_t)(q * 32) << 16;
        uint32_t norm_phase = 0;
        int it = 0;
        int sat = 0;
        int ovf = 0;                                // activations saturated to the fp16 range
        int wround = 0;                             // per-warp staging: rounds this warp has stored
        // GDN / IGDN with per-warp staging of one 32-channel round (BN = 128): a tile's y is staged
        // into the warp's slot right away, but its bulk tensor store -- whose issue stalls on the
        // TMA queue for ~1-2k cycles -- is issued while the NEXT tile waits for its norm MMAs
        // (DESIGN.md §7); d_* hold the deferred store's coordinates
        const bool defer = GC == 2 && p.wst_ch == 32 && p.wst_slots == 1;
        bool d_pending = false;
        int d_cb = 0, d_x = 0, d_y = 0, d_b = 0, d_ph = 0;
        auto flush_deferred = [&]() {
            if (!d_pending) return;
            d_pending = false;
            fence_proxy_async_smem();                  // the slot's generic writes -> the async proxy
            __syncwarp();
            if (lane == 0) {
                const uint8_t* hs = smem + p.off_ostage + (uint32_t)(warp - 4) * 4096u;
                if (p.nphase == 1) {
                    tma_store_5d(&mapOH, hs, d_cb, d_x, d_y, d_b, 0);
                } else {
                    const CUtensorMap* om = d_ph == 0 ? &mapOH : d_ph == 1 ? &mapOL : d_ph == 2 ? &mapO2 : &mapO3;
                    tma_store_4d(om, hs, d_cb, d_x, d_y, 0);
                }
                bulk_commit();
            }
        };
        // ---- two-group GDN / IGDN epilogue (p.g2, BN = 128): group gr = (warp - 4) / 8
        // takes this CTA's tiles it = gr, gr + 2, ... (accumulator buffer gr); warp (q, h) of the group
        // owns pixels 32q .. 32q + 31 (TMEM lanes) x channels 64h .. 64h + 63.  P1: x = acc + b, the
        // norm operand v = x^2 2^-2k (|x| 2^-k for 1DN; k per pixel, v_max in [2^13, 2^15)) as fp16
        // hi / lo written over the accumulator, the signs of x kept as bits; the MMA warp issues the
        // norm MMAs; P2: y from v and the norm alone -- x = sign sqrt(v) 2^k, so
        // y = x / sqrt(n) = sign v rsqrt(v n) 2^k (GDN), sign (v n) rsqrt(v n) 2^k (IGDN), one MUFU
        // op per value, and no register holds x across the norm round trip, during which the other
        // group works.
        if constexpr (GC == 2 || GC == 3) if (g2) {
            // NSUB 32-channel sub-blocks per thread (BN = 64 NSUB); BN = 192: the norm is computed in
            // three 64-column N chunks (chunk j = sub-block j of both channel halves: gamma rows 32j..
            // of each CTA's half), so a buffer is 192 accumulator + 64 norm columns and two fit in TMEM
            constexpr int NSUB = GC;
            constexpr bool kChunked = NSUB == 3;
            constexpr int CPT = 32 * NSUB;                            // channels per thread
            const int gr = (warp - 4) >> 3;
            const int h = ((warp - 4) >> 2) & 1;
            const int lead = 128 + gr * 256;                          // the group's first thread
            const uint32_t bar_full = 2u + (uint32_t)gr, bar_norm = 13u + (uint32_t)gr;
            const uint32_t bar_px = 5u + (uint32_t)(gr * 4 + q);      // the pixel's two channel halves
            const float s255 = p.l1_int ? (1.0f / 255.0f) : 1.0f;
            const uint32_t xe_a = s_xe + (uint32_t)(gr * 512) + 4u * (uint32_t)r;
            // per-warp output staging slot: rounds of wst = 32 (4 KB slots, 64-byte rows, 64B swizzle)
            // or 16 channels (2 KB slots, 32-byte rows, 32B swizzle: layers with 32 KB of staging)
            const bool w32 = p.wst_ch == 32;
            const uint32_t rows_b = w32 ? 64u : 32u, slot_b = 32u * rows_b * 2u, lo_off = 32u * rows_b;
            const uint32_t sw_mask = rows_b / 16u - 1u;
            // 16-channel rounds in two alternating 2 KB slots per warp (p.wst_slots == 2): a slot is
            // rewritten two rounds after its store was issued (wait_group.read 1, not 0)
            const bool db16 = !w32 && p.wst_slots == 2;
            const uint32_t slot_off0 = p.off_ostage + (uint32_t)(warp - 4) * slot_b * (db16 ? 2u : 1u);
            const uint32_t sw = (((uint32_t)lane * rows_b) >> 7) & sw_mask;     // swizzle of this row
            const int ty0 = (q * 32) >> p.wt_log2, tx0 = (q * 32) & (p.Wt - 1);
            const uint32_t tbuf = tmem_base + lane_off + (uint32_t)(gr * p.acc_stride);
            const uint32_t tcol0 = tbuf + (uint32_t)(h * CPT);
            // this thread's norm columns: the whole norm region (NSUB = 2) or its 32 of a chunk's 64
            const uint32_t tnorm = kChunked ? tbuf + (uint32_t)p.BN + (uint32_t)(32 * h) : tcol0 + (uint32_t)p.BN;
            const int c0 = h * CPT;                                    // first channel of this thread (one N tile)
            bool gamma_ok = false;                                     // (the norm-issuing thread) gamma landed
            // |bias| bound of this thread's channels: max |x| <= max |acc| s255 + bmax (the exponent
            // below is taken from this bound, so the accumulator is read once before the exchange)
            float bmax = 0.0f;
            for (int i = 0; i < CPT; ++i) bmax = fmaxf(bmax, fabsf(s_bias[c0 + i]));
            // norm MMAs of chunk j (all of them for NSUB = 2), issued by the leader's group-lead thread
            auto issue_norm_g2 = [&](int j) {
                const uint32_t dcol = (uint32_t)(gr * p.acc_stride);
                const uint32_t ncol = tmem_base + dcol + (uint32_t)p.BN;
                const uint32_t gbase = smem_u32(smem + p.off_gamma) + (kChunked ? (uint32_t)(j * 32 * 128) : 0u);
                const uint32_t nn = kChunked ? 64u : (uint32_t)p.BN;
                const uint32_t idesc_n = idesc_f16_f32(kBM * CG, nn);
#pragma unroll
                for (int kk = 0; kk < 4 * NSUB; ++kk) {   // K = BN in steps of 16 (G = 32 layout)
                    const int k0 = 16 * kk, gg = k0 / 32, o = k0 - gg * 32;
                    const uint32_t ahi = tmem_base + dcol + gg * 32 + o / 2;
                    const uint64_t bd = sdesc_sw128(gbase + (k0 / 64) * (uint32_t)((p.BN / CG) * kBK * 2)) + 2 * (kk & 3);
                    if constexpr (CG == 2) {
                        umma_f16_ts_cg2(ncol, ahi, bd, idesc_n, kk != 0);
                        umma_f16_ts_cg2(ncol, ahi + 16, bd, idesc_n, 1u);
                    } else {
                        umma_f16_ts(ncol, ahi, bd, idesc_n, kk != 0);
                        umma_f16_ts(ncol, ahi + 16, bd, idesc_n, 1u);
                    }
                }
                if constexpr (CG == 2) umma_commit_pair(&norm2_bar[gr]); else umma_commit(&norm2_bar[gr]);
            };
            auto arrive_group = [&]() {          // this warp is done with v / the norm chunk (leader's barrier)
                tc_fence_before();
                __syncwarp();
                if (lane == 0) {
                    if constexpr (CG == 2) mbar_arrive_cluster(lbar(&xsq2_bar[gr]));
                    else mbar_arrive(&xsq2_bar[gr]);
                }
            };
            auto body = [&](auto onedn_c, auto fwd_c) {
                constexpr bool kOneDN = decltype(onedn_c)::value, kFwd = decltype(fwd_c)::value;
                int it = gr;
                for (int t = cid + gr * ncl; t < p.total_tiles; t += 2 * ncl, it += 2) {
                    const TileCoord tc = decode_tile<kSplitK>(p, t, rank);
                    const uint32_t par = (uint32_t)(it >> 1) & 1u;
                    // barrier phases per tile: xsq2 / norm2 complete once per tile (NSUB = 2) or once
                    // per norm chunk (3 per tile): phase number ph0 + j
                    const uint32_t ph0 = kChunked ? 3u * (uint32_t)(it >> 1) : (uint32_t)(it >> 1);
                    const bool tma_ok = p.nphase == 1 || tc.gy0 + ty0 + 32 / (p.Wt < 32 ? p.Wt : 32) <= p.Hg;
                    const bool slow = !tma_ok || p.out_f32 != nullptr;
                    if (threadIdx.x == lead) mbar_wait(&tfull_bar[gr], par);
                    named_bar_sync(bar_full, 256);
                    tc_fence_after();
                    if (threadIdx.x == lead) LIC_TRACE(it, T_EPI_START);
                    // ---- P1.  Pass A: a bound on max |x| of the pixel (both channel halves);
                    // pass B, 32 channels at a time: x = acc s255 + b, v, signs, v -> TMEM.
                    uint32_t xr[32];
                    float amax = 0.0f;
#pragma unroll 1
                    for (int s = 0; s < NSUB; ++s) {
                        tmem_ld32_nw(tcol0 + 32 * s, xr);
                        tmem_ld_wait_dep32(xr);
#pragma unroll
                        for (int i = 0; i < 32; ++i) amax = fmaxf(amax, fabsf(__uint_as_float(xr[i])));
                    }
                    const float xb = fmaf(amax, s255, bmax);
                    stsb(xe_a + (uint32_t)h, __float_as_uint(xb) >> 23);        // biased exponent of the bound
                    named_bar_sync(bar_px, 64);
                    const uint32_t ew = ldsu(xe_a);
                    const int E = (int)max(ew & 0xffu, (ew >> 8) & 0xffu) - 127;   // max |x| < 2^(E+1)
                    // GDN: v = x^2 2^-2k, k = E - 6 -> v < 2^14; 1DN: v = |x| 2^-k, k = E - 13 -> v < 2^14
                    const int k = kOneDN ? min(max(E - 13, -100), 100) : min(max(E - 6, -50), 50);
                    const float sc_dn = __int_as_float((127 - k) << 23);          // 2^-k
                    uint32_t sg0 = 0u, sg1 = 0u, sg2 = 0u;                   // sign bits (bit 31 = channel 32s)
#pragma unroll 1
                    for (int s = 0; s < NSUB; ++s) {
                        tmem_ld32_nw(tcol0 + 32 * s, xr);
                        tmem_ld_wait_dep32(xr);
                        uint32_t hv[16], lv[16];
                        uint32_t sgs = 0u;
#pragma unroll
                        for (int i4 = 0; i4 < 8; ++i4) {
                            const float4 bb = lds4(s_bias + c0 + 32 * s + 4 * i4);
                            const float bq[4] = {bb.x, bb.y, bb.z, bb.w};
                            float v[4];
#pragma unroll
                            for (int u = 0; u < 4; ++u) {
                                const float xv = fmaf(__uint_as_float(xr[4 * i4 + u]), s255, bq[u]);
                                sgs = __funnelshift_l(__float_as_uint(xv), sgs, 1);   // (sgs << 1) | sign
                                const float xs = xv * sc_dn;                  // x 2^-k (GDN), |x| 2^-k (1DN)
                                v[u] = kOneDN ? fabsf(xs) : xs * xs;
                            }
                            split2(v[0], v[1], hv[2 * i4], lv[2 * i4]);
                            split2(v[2], v[3], hv[2 * i4 + 1], lv[2 * i4 + 1]);
                        }
                        if (s == 0) sg0 = sgs; else if (s == 1) sg1 = sgs; else sg2 = sgs;
                        // the G = 32 layout of the norm MMA: hi of channel 32s + j at column 32s + j/2, lo at 32s + 16 + j/2
                        const uint32_t ts = tcol0 + 32u * (uint32_t)s;
                        tmem_st8(ts, hv);
                        tmem_st8(ts + 8, hv + 8);
                        tmem_st8(ts + 16, lv);
                        tmem_st8(ts + 24, lv + 8);
                    }
                    tmem_st_wait();
                    arrive_group();
                    if (threadIdx.x == lead) LIC_TRACE(it, T_EPI_XSQ);
                    if (leader && threadIdx.x == lead) {
                        // every warp of the group (both CTAs) has written v: issue norm = v . gamma^T
                        // from here (a blocking wait: the MMA warp keeps issuing main loops meanwhile)
                        if (!gamma_ok) { mbar_wait(gamma_bar, 0); gamma_ok = true; }
                        mbar_wait(&xsq2_bar[gr], ph0 & 1u);
                        tc_fence_after();
                        issue_norm_g2(0);
                    }
                    // ---- wait for the norm MMAs of this tile (NSUB = 3: of chunk 0; later chunks in P2)
                    auto wait_norm = [&](int j) {
                        if (threadIdx.x == lead) mbar_wait(&norm2_bar[gr], (ph0 + (uint32_t)j) & 1u);
                        named_bar_sync(bar_norm, 256);
                        tc_fence_after();
                    };
                    wait_norm(0);
                    if (threadIdx.x == lead) LIC_TRACE(it, T_EPI_NORM);
                    // n = beta + c 2^(2k) (GDN) / beta + c 2^k (1DN), c the contraction of v
                    const float sc_up = kOneDN ? __int_as_float((127 + k) << 23) : __int_as_float((127 + 2 * k) << 23);
                    const float sc_k = __int_as_float((127 + k) << 23);       // |x| = sqrt(v) 2^k (GDN), v 2^k (1DN)
                    // ---- P2: 2 NSUB pieces of 16 channels; pieces 2s, 2s + 1 form staging round s (32
                    // channels) -- and, chunked, norm chunk s
#pragma unroll 1
                    for (int pc = 0; pc < 2 * NSUB; ++pc) {
                        const int j = pc & 1;
                        if (kChunked && j == 0 && pc > 0) wait_norm(pc >> 1);
                        const uint32_t slot_off = slot_off0 + (db16 ? (uint32_t)(pc & 1) * slot_b : 0u);
                        const uint32_t rowa = smem_u32(smem) + slot_off + (uint32_t)lane * rows_b;
                        if (j == 0 || !w32) {
                            if (lane == 0 && !(p.dbg_nostore & 128)) { if (db16) bulk_wait_read1(); else bulk_wait_read0(); }   // the slot is free again
                            __syncwarp();
                        }
                        uint32_t vh[8], vl[8], nr[16];
                        const uint32_t ts = tcol0 + 32u * (uint32_t)(pc >> 1) + 8u * (uint32_t)j;
                        tmem_ld8_nw(ts, vh);
                        tmem_ld8_nw(ts + 16, vl);
                        tmem_ld16_nw(kChunked ? tnorm + 16u * (uint32_t)j : tnorm + 16u * (uint32_t)pc, nr);
                        tmem_ld_wait_dep(vh, vl, nr);
                        if (kChunked && j == 1 && pc < 2 * NSUB - 1) {
                            // this warp has read norm chunk s: the lead thread may overwrite the region
                            // with chunk s + 1 once every warp of the group (both CTAs) has
                            arrive_group();
                            if (leader && threadIdx.x == lead) {
                                mbar_wait(&xsq2_bar[gr], (ph0 + (uint32_t)(pc >> 1) + 1u) & 1u);
                                tc_fence_after();
                                issue_norm_g2((pc >> 1) + 1);
                            }
                        }
                        if (pc == 2 * NSUB - 1) {
                            // every TMEM read of this tile is complete: release the buffer
                            tc_fence_before();
                            __syncwarp();
                            if (lane == 0) {
                                if constexpr (CG == 2) mbar_arrive_cluster(lbar(&tempty_bar[gr]));
                                else mbar_arrive(&tempty_bar[gr]);
                            }
                        }
                        const uint32_t sgw = (pc >> 1) == 0 ? sg0 : (pc >> 1) == 1 ? sg1 : sg2;
                        const uint32_t sgp = sgw << (16 * j);          // bit 31 = this piece's channel 0
                        float y[16];
#pragma unroll
                        for (int i4 = 0; i4 < 4; ++i4) {
                            const float4 be = lds4(s_beta + c0 + 16 * pc + 4 * i4);
                            const float bv[4] = {be.x, be.y, be.z, be.w};
#pragma unroll
                            for (int u = 0; u < 4; ++u) {
                                const int i = 4 * i4 + u;
                                const float v = (i & 1) ? join_h<1>(vh[i >> 1], vl[i >> 1]) : join_h<0>(vh[i >> 1], vl[i >> 1]);
                                const float nn = fmaf(__uint_as_float(nr[i]), sc_up, bv[u]);
                                float m;
                                if constexpr (kOneDN) {
                                    m = kFwd ? (v * sc_k) * rcp_ftz(nn) : (v * sc_k) * nn;    // |x| / n, |x| n
                                } else {
                                    const float tv = fmaf(v, nn, 1e-30f);                    // v = 0: y = 0
                                    const float rs = rsqrt_ftz(tv);
                                    m = (kFwd ? v * rs : tv * rs) * sc_k;     // |x| / sqrt(n), |x| sqrt(n)
                                }
                                y[i] = __uint_as_float(__float_as_uint(m) ^ ((sgp << i) & 0x80000000u));
                            }
                        }
                        if (slow) {
                            // test-only f32 copy, and a transposed conv's tile crossing the grid's bottom
                            // edge (the phase view would run into the next frame): direct stores
                            const int gy = tc.gy0 + (r >> p.wt_log2), gx = tc.gx0 + (r & (p.Wt - 1));
                            const bool valid = gy < p.Hg && gx < p.Wg;
                            const int oy = p.out_s * gy + (p.nphase == 4 ? (tc.ph >> 1) : 0);
                            const int ox = p.out_s * gx + (p.nphase == 4 ? (tc.ph & 1) : 0);
                            const int cb = tc.nt * p.BN + c0 + 16 * pc;
                            if (p.out_f32 && valid) {
                                const size_t HWo = (size_t)p.Hout * p.Wout;
                                const size_t chw0 = (size_t)tc.b * p.Cout * HWo + (size_t)oy * p.Wout + ox;
#pragma unroll
                                for (int i = 0; i < 16; ++i) p.out_f32[chw0 + (size_t)(cb + i) * HWo] = y[i];
                            }
                            if (!tma_ok) {
                                guard16(y, ovf);
                                if (valid) {
                                    __half* out = reinterpret_cast<__half*>(p.out_act);
                                    const size_t pix = ((size_t)tc.b * p.Hout + oy) * p.Wout + ox;
                                    split_store8(out + pix * p.Cout + cb, out + p.act_plane + pix * p.Cout + cb, y);
                                    split_store8(out + pix * p.Cout + cb + 8, out + p.act_plane + pix * p.Cout + cb + 8, y + 8);
                                }
                                continue;
                            }
                        }
                        if (!p.no_guard) guard16(y, ovf);
                        if (p.dbg_nostore & 64) {                   // experiment (traced layer): compute only
                            if (lane == 0 && __float_as_uint(y[0] + y[15]) == 0x7fc00001u) p.out_f32[0] = y[1];
                            continue;
                        }
#pragma unroll
                        for (int kk = 0; kk < 2; ++kk) {
                            uint4 hq, lq;
                            const float* v8 = y + 8 * kk;
                            split2(v8[0], v8[1], hq.x, lq.x); split2(v8[2], v8[3], hq.y, lq.y);
                            split2(v8[4], v8[5], hq.z, lq.z); split2(v8[6], v8[7], hq.w, lq.w);
                            const uint32_t o = ((((uint32_t)((w32 ? 2 * j : 0) + kk)) ^ sw) & sw_mask) << 4;
                            stsu4(rowa + o, hq);
                            stsu4(rowa + lo_off + o, lq);
                        }
                        if (j == 1 || !w32) {
                            fence_proxy_async_smem();
                            __syncwarp();
                            if (lane == 0) {
                                if (threadIdx.x == lead) LIC_TRACE(it, pc == 2 * NSUB - 1 ? T_EPI_ACQ : T_EPI_P2);
                                const uint8_t* hs = smem + slot_off;
                                const int cb = tc.nt * p.BN + c0 + (w32 ? 32 * (pc >> 1) : 16 * pc);
                                if (p.dbg_nostore & 32) {                   // experiment (traced layer): no TMA store
                                } else if (p.nphase == 1) {
                                    tma_store_5d(&mapOH, hs, cb, tc.gx0 + tx0, tc.gy0 + ty0, tc.b, 0);
                                } else {
                                    const int ph = tc.ph;
                                    const CUtensorMap* om = ph == 0 ? &mapOH : ph == 1 ? &mapOL : ph == 2 ? &mapO2 : &mapO3;
                                    tma_store_4d(om, hs, cb, tc.gx0 + tx0, tc.b * p.Hg + tc.gy0 + ty0, 0);
                                }
                                bulk_commit();
                                if (threadIdx.x == lead) LIC_TRACE(it, pc == 2 * NSUB - 1 ? T_EPI_END : T_EPI_STAGED);
                            }
                        }
                    }
                }
            };
            using T_ = std::integral_constant<bool, true>;
            using F_ = std::integral_constant<bool, false>;
            if (p.onedn) { if (p.ep == EP_GDN) body(T_{}, T_{}); else body(T_{}, F_{}); }
            else { if (p.ep == EP_GDN) body(F_{}, T_{}); else body(F_{}, F_{}); }
        }
        for (int t = g2 ? p.total_tiles : cid; t < p.total_tiles; t += ncl, ++it) {
            TileCoord tc = decode_tile<kSplitK>(p, t, rank);
            const int buf = (p.n_accbuf == 2) ? (it & 1) : 0;
            const uint32_t use = (p.n_accbuf == 2) ? (uint32_t)(it >> 1) : (uint32_t)it;
            // one lane waits on the mbarrier, the other epilogue warps sleep in a hardware
            // named barrier (no polling: keeps the SYNCS unit and the issue slots free)
            if (threadIdx.x == 128) mbar_wait(&tfull_bar[buf], use & 1);
            named_bar_sync(2, 32 * kEpiWarps);
            tc_fence_after();
            if (threadIdx.x == 128) LIC_TRACE(it, T_EPI_START);
            const uint32_t dcol = (uint32_t)(buf * p.acc_stride);
            const uint32_t taddr = tmem_base + lane_off + dcol;

            const int gy = tc.gy0 + (r >> p.wt_log2), gx = tc.gx0 + (r & (p.Wt - 1));
            const bool valid = (gy < p.Hg) && (gx < p.Wg);
            const int py = (p.nphase == 4) ? (tc.ph >> 1) : 0;
            const int px = (p.nphase == 4) ? (tc.ph & 1) : 0;
            const int oy = p.out_s * gy + py, ox = p.out_s * gx + px;
            const size_t pix = ((size_t)tc.b * p.Hout + oy) * p.Wout + ox;
            const size_t HWo = (size_t)p.Hout * p.Wout;
            const size_t chw0 = (size_t)tc.b * p.Cout * HWo + (size_t)oy * p.Wout + ox;
            const int co0 = tc.nt * p.BN;
            // this warp's 32 pixels form a bw x bh box at tile offset (tx0, ty0)
            const int bw = p.Wt < 32 ? p.Wt : 32, bh = 32 / bw;
            const int ty0 = (q * 32) >> p.wt_log2, tx0 = (q * 32) & (p.Wt - 1);
            const bool tma_ok = p.tma_out && (p.nphase == 1 || tc.gy0 + ty0 + bh <= p.Hg);
            // TMA-store staging, per TMEM lane quadrant: the quadrant's 4 warps (channel groups)
            // fill 64-channel blocks of their 32 pixels -- [plane hi | lo][32 px][128 B], 128B-
            // swizzled (16-byte piece c of row r at ((c ^ (r & 7)) << 4): conflict-free 16-byte
            // stores) -- in p.ostage_slots 8 KB slots; one elected thread per quadrant then stores
            // each block with one bulk tensor store per plane (128-byte rows: 4x fewer TMA
            // requests than 16-channel boxes).
            const int qslots = p.ostage_slots;
            const uint32_t qstage = smem_u32(smem + p.off_ostage) + (uint32_t)(q * qslots * 8192);
            const bool qissuer = (g == 0) && (lane == 0);
            auto stage16 = [&](const float* v16, int cb, int slot) {
                uint4 h0, h1, l0, l1;
                split2(v16[0], v16[1], h0.x, l0.x);   split2(v16[2], v16[3], h0.y, l0.y);
                split2(v16[4], v16[5], h0.z, l0.z);   split2(v16[6], v16[7], h0.w, l0.w);
                split2(v16[8], v16[9], h1.x, l1.x);   split2(v16[10], v16[11], h1.y, l1.y);
                split2(v16[12], v16[13], h1.z, l1.z); split2(v16[14], v16[15], h1.w, l1.w);
                if (p.dbg_nostore & 16) return;                                   // experiment: no staging writes
                const uint32_t base = qstage + (uint32_t)slot * 8192u + (uint32_t)lane * 128u;
                const uint32_t c0 = (uint32_t)((cb & 63) >> 3);                 // 16-byte piece of channel cb
                const uint32_t o0 = ((c0 ^ (uint32_t)(lane & 7)) << 4), o1 = (((c0 + 1) ^ (uint32_t)(lane & 7)) << 4);
                stsu4(base + o0, h0);
                stsu4(base + o1, h1);
                stsu4(base + 4096u + o0, l0);
                stsu4(base + 4096u + o1, l1);
            };
            // every thread of the quadrant: slots free (the issuer waited for their previous stores
            // to finish reading smem; `keep` groups may stay in flight)
            auto q_acquire = [&](int keep) {
                if (qissuer) { if (keep) bulk_wait_read1(); else bulk_wait_read0(); }
                named_bar_sync(5 + q, 128);
            };
            // blocks [blk0, blk0 + nblk) are in slots 0.. : make them visible and store them
            auto q_flush = [&](int blk0, int nblk, int slot0) {
                fence_proxy_async_smem();
                named_bar_sync(5 + q, 128);
                if (qissuer && !(p.dbg_nostore & 8)) {                               // 8: experiment, no TMA
                    for (int k = 0; k < nblk; ++k) {
                        const uint8_t* os = smem + p.off_ostage + (size_t)(q * qslots + slot0 + k) * 8192u;
                        const int cb = co0 + 64 * (blk0 + k);
                        if (p.nphase == 1) {
                            tma_store_4d(&mapOH, os, cb, tc.gx0 + tx0, tc.gy0 + ty0, tc.b);
                            if (p.split == 2) tma_store_4d(&mapOL, os + 4096, cb, tc.gx0 + tx0, tc.gy0 + ty0, tc.b);
                        } else {
                            const int qyb = tc.b * p.Hg + tc.gy0 + ty0;
                            tma_store_5d(&mapOH, os, cb, px, tc.gx0 + tx0, py, qyb);
                            if (p.split == 2) tma_store_5d(&mapOL, os + 4096, cb, px, tc.gx0 + tx0, py, qyb);
                        }
                    }
                    bulk_commit();
                }
            };
            auto direct16 = [&](const float* v16, int cb) {
                __half* out = reinterpret_cast<__half*>(p.out_act);
                if (!valid) return;
                split_store8(out + pix * p.Cout + cb, p.split == 2 ? out + p.act_plane + pix * p.Cout + cb : nullptr, v16);
                split_store8(out + pix * p.Cout + cb + 8, p.split == 2 ? out + p.act_plane + pix * p.Cout + cb + 8 : nullptr,
                             v16 + 8);
            };
            // generic epilogues: round k of the channel loop holds block k (warp g: channels
            // 64k + 16g ..) -- one block per round through alternating slots
            auto emit16 = [&](float* v16, int cb) {
                guard16(v16, ovf);
                if (!tma_ok) { direct16(v16, cb); return; }
                const int blk = (cb - co0) >> 6, slot = blk % qslots;
                q_acquire(qslots - 1);
                stage16(v16, cb - co0, slot);
                q_flush(blk, 1, slot);
            };
            bool released = false;
            if constexpr (kGdn) {
                constexpr int G = 16 * GC;                   // channels of this group
                float x[GC][16];
                __syncwarp();
#pragma unroll
                for (int j = 0; j + 1 < GC; j += 2) tmem_ld32(taddr + g * G + j * 16, x[j]);
                if constexpr (GC & 1) tmem_ld16(taddr + g * G + (GC - 1) * 16, x[GC - 1]);
                // x = acc (/ 255 for integer u8 samples) + b, and the largest norm operand v of the
                // pixel (v = x^2, or |x| for 1DN) over this group's channels
                float vmax = 0.0f;
#pragma unroll
                for (int j = 0; j < GC; ++j) {
                    if (p.l1_int) {
                        // fused g_a L1 on u8 samples: acc = sum W * u exactly; x = acc / 255 + b
#pragma unroll
                        for (int i = 0; i < 16; ++i) x[j][i] *= (1.0f / 255.0f);
                    }
#pragma unroll
                    for (int i4 = 0; i4 < 4; ++i4) {
                        const float4 bb = lds4(s_bias + g * G + j * 16 + 4 * i4);
                        x[j][4 * i4 + 0] += bb.x; x[j][4 * i4 + 1] += bb.y;
                        x[j][4 * i4 + 2] += bb.z; x[j][4 * i4 + 3] += bb.w;
                    }
#pragma unroll
                    for (int i = 0; i < 16; ++i)
                        vmax = fmaxf(vmax, p.onedn ? fabsf(x[j][i]) : x[j][i] * x[j][i]);
                }
                // The norm operand goes to the tensor core as fp16 hi + lo, whose range ends at
                // 65504 (x^2 overflows from |x| = 256 on).  Every pixel scales its operand by
                // 2^-e, e = the smallest shift that keeps the pixel's largest v below 2^15 (0 for
                // v < 2^14: the common case is unscaled, bit for bit), and the epilogue multiplies
                // the contraction by 2^e -- both exact.  e is shared by the pixel's 4 channel
                // groups (one byte each in smem, max over the quadrant's 4 warps).
                {
                    const int ex = (__float_as_int(vmax) >> 23) - 127;
                    stsb(s_xe + 4u * (uint32_t)r + (uint32_t)g, (uint32_t)min(max(ex - 13, 0), 100));
                }
                named_bar_sync(5 + q, 128);
                uint32_t xe = ldsu(s_xe + 4u * (uint32_t)r);
                xe = max(max(xe & 0xffu, (xe >> 8) & 0xffu), max((xe >> 16) & 0xffu, xe >> 24));
                const float sc_dn = __int_as_float((int)(127u - xe) << 23);
                const float sc_up = __int_as_float((int)(127u + xe) << 23);
                // v * 2^-e (hi, lo) packed into this group's own accumulator columns:
                // hi of channel g*G + k at column g*G + k/2, lo at g*G + G/2 + k/2
#pragma unroll
                for (int j = 0; j < GC; ++j) {
                    uint32_t hi[8], lo[8];
                    if (p.onedn) {
#pragma unroll
                        for (int i = 0; i < 8; ++i)
                            split2(fabsf(x[j][2 * i]) * sc_dn, fabsf(x[j][2 * i + 1]) * sc_dn, hi[i], lo[i]);
                    } else {
#pragma unroll
                        for (int i = 0; i < 8; ++i) {
                            const float a2 = x[j][2 * i] * x[j][2 * i], b2 = x[j][2 * i + 1] * x[j][2 * i + 1];
                            split2(a2 * sc_dn, b2 * sc_dn, hi[i], lo[i]);
                        }
                    }
                    tmem_st8(taddr + g * G + j * 8, hi);
                    tmem_st8(taddr + g * G + G / 2 + j * 8, lo);
                }
                tmem_st_wait();
                tc_fence_before();
                __syncwarp();
                if (lane == 0) {
                    // the (leader's) MMA warp issues the norm MMAs
                    if constexpr (CG == 2) {
                        mbar_arrive_cluster(lbar(xsq_bar));
                        atom_add_cluster(mapa_shared(smem_u32(xsq_cnt), 0), 1u);
                    } else {
                        mbar_arrive(xsq_bar);
                        atomicAdd(xsq_cnt, 1u);
                    }
                }
                if (threadIdx.x == 128) LIC_TRACE(it, T_EPI_XSQ);
                if (defer) flush_deferred();             // the previous tile's y, under the norm MMAs
                if (threadIdx.x == 128) mbar_wait(norm_bar, norm_phase);
                norm_phase ^= 1;
                named_bar_sync(3, 32 * kEpiWarps);
                tc_fence_after();
                if (threadIdx.x == 128) LIC_TRACE(it, T_EPI_NORM);
                __half* out = reinterpret_cast<__half*>(p.out_act);
                // GC = 2: both norm column blocks in flight at once (one TMEM wait); GC = 3
                // loads them one by one (three at once would spill)
                constexpr int kNB = GC == 2 ? 2 : 1;
                float nall[kNB][16];
                if constexpr (GC == 2) {
                    __syncwarp();
                    tmem_ld32(taddr + p.BN + g * G, nall[0]);
                }
#pragma unroll
                for (int j = 0; j < GC; ++j) {
                    float* n = nall[GC == 2 ? j : 0];
                    if constexpr (GC != 2) {
                        __syncwarp();
                        tmem_ld16(taddr + p.BN + g * G + j * 16, n);
                    }
                    if (p.dbg_nostore & 4) {
#pragma unroll
                        for (int i = 0; i < 16; ++i) n[i] = x[j][i];
                    }
                    const int cb = g * G + j * 16;
#pragma unroll
                    for (int i4 = 0; i4 < 4; ++i4) {
                        const float4 be = lds4(s_beta + cb + 4 * i4);
                        const float bv[4] = {be.x, be.y, be.z, be.w};
                        if (p.onedn) {
                            // 1DN: y = x / n (forward), x * n (inverse); n = beta + gamma |x|
#pragma unroll
                            for (int u = 0; u < 4; ++u) {
                                const int i = 4 * i4 + u;
                                const float nn = bv[u] + n[i] * sc_up;
                                x[j][i] = (p.ep == EP_GDN) ? x[j][i] * rcp_ftz(nn) : x[j][i] * nn;
                            }
                        } else {
#pragma unroll
                            for (int u = 0; u < 4; ++u) {
                                const int i = 4 * i4 + u;
                                const float nn = bv[u] + n[i] * sc_up;
                                const float rs = (p.dbg_nostore & 2) ? nn : rsqrt_ftz(nn);   // MUFU; sqrt(nn) = nn * rsqrt(nn)
                                x[j][i] = (p.ep == EP_GDN) ? x[j][i] * rs : x[j][i] * (nn * rs);
                            }
                        }
                    }
                    if (valid && p.out_f32) {
#pragma unroll
                        for (int i = 0; i < 16; ++i) p.out_f32[chw0 + (size_t)(cb + i) * HWo] = x[j][i];
                    }
                    guard16(x[j], ovf);
                }
                if (threadIdx.x == 128) LIC_TRACE(it, T_EPI_P2);
                // the accumulator is in registers: release TMEM before storing
                tc_fence_before();
                __syncwarp();
                if (lane == 0) {
                    if constexpr (CG == 2) mbar_arrive_cluster(lbar(&tempty_bar[buf]));
                    else mbar_arrive(&tempty_bar[buf]);
                }
                released = true;
                if (out && !(p.dbg_nostore & 1)) {
                    if (defer && tma_ok) {
                        // stage now (the slot's previous store has been issued and read), store
                        // during the next tile's norm wait (or at the end)
                        const uint32_t rows_b = 64u;
                        const uint32_t sw = (((uint32_t)lane * rows_b) >> 7) & 3u;
                        const uint32_t rowa = smem_u32(smem) + (uint32_t)p.off_ostage + (uint32_t)(warp - 4) * 4096u +
                                              (uint32_t)lane * rows_b;
                        if (lane == 0) bulk_wait_read0();
                        __syncwarp();
#pragma unroll
                        for (int j = 0; j < 2; ++j)
#pragma unroll
                            for (int k = 0; k < 2; ++k) {
                                uint4 hv, lv;
                                const float* v8 = x[j] + 8 * k;
                                split2(v8[0], v8[1], hv.x, lv.x); split2(v8[2], v8[3], hv.y, lv.y);
                                split2(v8[4], v8[5], hv.z, lv.z); split2(v8[6], v8[7], hv.w, lv.w);
                                const uint32_t o = ((((uint32_t)(2 * j + k)) ^ sw) & 3u) << 4;
                                stsu4(rowa + o, hv);
                                if (p.split == 2) stsu4(rowa + 32u * rows_b + o, lv);
                            }
                        d_cb = co0 + g * G;
                        d_ph = py * 2 + px;
                        d_x = tc.gx0 + tx0;
                        d_y = p.nphase == 1 ? tc.gy0 + ty0 : tc.b * p.Hg + tc.gy0 + ty0;
                        d_b = tc.b;
                        d_pending = true;
                    } else if (tma_ok && p.wst_ch) {
                        // per-warp staging: this warp's 32 pixels x its G channels in
                        // rounds of wst_ch channels (rows of 2 * wst_ch bytes, swizzled like the
                        // out maps), each round written by the warp's own bulk tensor stores --
                        // no cross-warp barrier; wst_slots slots per warp, reused round-robin
                        const int rch = p.wst_ch, per = rch / 16, nsl = p.wst_slots;
                        const uint32_t rows_b = 2u * (uint32_t)rch, slot_bytes = 128u * (uint32_t)rch;
                        const uint32_t sw_mask = rows_b / 16u - 1u;
                        const uint32_t sw = (((uint32_t)lane * rows_b) >> 7) & sw_mask;
                        const uint32_t wbase = (uint32_t)p.off_ostage + (uint32_t)(warp - 4) * (uint32_t)nsl * slot_bytes;
                        if (threadIdx.x == 128) LIC_TRACE(it, T_EPI_ACQ);
#pragma unroll
                        for (int j = 0; j < GC; ++j) {
                            const int kk = j % per;
                            const uint32_t sl = wbase + (uint32_t)(wround % nsl) * slot_bytes;
                            if (kk == 0) {
                                // the stores nsl rounds ago (same slot) have read it
                                if (lane == 0) { if (nsl == 2) bulk_wait_read1(); else bulk_wait_read0(); }
                                __syncwarp();
                            }
                            if (threadIdx.x == 128 && !p.fuse_l1 && j == 0) LIC_TRACE(it, T_B_PATCH);
                            const uint32_t rowa = smem_u32(smem) + sl + (uint32_t)lane * rows_b;
#pragma unroll
                            for (int k = 0; k < 2; ++k) {                    // 16-byte chunks (8 channels)
                                uint4 hv, lv;
                                const float* v8 = x[j] + 8 * k;
                                split2(v8[0], v8[1], hv.x, lv.x); split2(v8[2], v8[3], hv.y, lv.y);
                                split2(v8[4], v8[5], hv.z, lv.z); split2(v8[6], v8[7], hv.w, lv.w);
                                const uint32_t o = ((((uint32_t)(2 * kk + k)) ^ sw) & sw_mask) << 4;
                                stsu4(rowa + o, hv);
                                if (p.split == 2) stsu4(rowa + 32u * rows_b + o, lv);
                            }
                            if (kk == per - 1 || j == GC - 1) {
                                if (threadIdx.x == 128 && !p.fuse_l1 && j == GC - 1) LIC_TRACE(it, T_B_C0_READY);
                                fence_proxy_async_smem();
                                __syncwarp();
                                if (threadIdx.x == 128 && !p.fuse_l1 && j == GC - 1) LIC_TRACE(it, T_B_C0_DONE);
                                if (lane == 0) {
                                    // one store writes both planes (the map's last dimension)
                                    const int cb = co0 + g * G + 16 * (j - kk);
                                    const uint8_t* hs = smem + sl;
                                    if (p.nphase == 1) {
                                        tma_store_5d(&mapOH, hs, cb, tc.gx0 + tx0, tc.gy0 + ty0, tc.b, 0);
                                    } else {
                                        const int ph = py * 2 + px;
                                        const CUtensorMap* om = ph == 0 ? &mapOH : ph == 1 ? &mapOL : ph == 2 ? &mapO2 : &mapO3;
                                        tma_store_4d(om, hs, cb, tc.gx0 + tx0, tc.b * p.Hg + tc.gy0 + ty0, 0);
                                    }
                                    bulk_commit();
                                }
                                ++wround;
                            }
                        }
                        if (threadIdx.x == 128) LIC_TRACE(it, T_EPI_STAGED);
                    } else if (tma_ok) {
                        const int nblk = p.BN >> 6;
                        for (int b0 = 0; b0 < nblk; b0 += qslots) {
                            q_acquire(0);
                            if (threadIdx.x == 128 && b0 == 0) LIC_TRACE(it, T_EPI_ACQ);
#pragma unroll
                            for (int j = 0; j < GC; ++j) {
                                const int cb = g * G + j * 16, blk = cb >> 6;
                                if (blk >= b0 && blk < b0 + qslots) stage16(x[j], cb, blk - b0);
                            }
                            if (threadIdx.x == 128 && b0 == 0) LIC_TRACE(it, T_EPI_STAGED);
                            q_flush(b0, min(qslots, nblk - b0), 0);
                        }
                    } else {
#pragma unroll
                        for (int j = 0; j < GC; ++j) direct16(x[j], g * G + j * 16);
                    }
                }
            } else if (!kL1 && p.gather) {
                // ---- gather mode (g_s L4): P[p][t][0..11] -> smem, then each output sums its 9
                // neighbours' slices.  Column chunk t (16 wide) of the accumulator = offset t.
                const uint32_t gp = smem_u32(smem + p.off_gp);
                for (int t9 = g; t9 < 9; t9 += kEpiGroups) {
                    float v[16];
                    __syncwarp();
                    tmem_ld16(taddr + t9 * 16, v);
                    const uint32_t row = gp + (uint32_t)((t9 * 128 + r) * 48);
                    // compact the 12 real columns (phase*4 + co, co < 3) to phase*3 + co
                    stsu4(row, make_uint4(__float_as_uint(v[0]), __float_as_uint(v[1]), __float_as_uint(v[2]),
                                          __float_as_uint(v[4])));
                    stsu4(row + 16, make_uint4(__float_as_uint(v[5]), __float_as_uint(v[6]), __float_as_uint(v[8]),
                                               __float_as_uint(v[9])));
                    stsu4(row + 32, make_uint4(__float_as_uint(v[10]), __float_as_uint(v[12]), __float_as_uint(v[13]),
                                               __float_as_uint(v[14])));
                }
                // accumulator consumed: release it, then gather once every warp has staged P
                tc_fence_before();
                __syncwarp();
                if (lane == 0) {
                    if constexpr (CG == 2) mbar_arrive_cluster(lbar(&tempty_bar[buf]));
                    else mbar_arrive(&tempty_bar[buf]);
                }
                released = true;
                named_bar_sync(3, 32 * kEpiWarps);
                // work item: output row (oy, py) = w / 28, column x = 2 ox + px = w % 28
                for (int w = threadIdx.x - 128; w < 6 * 2 * 28; w += 32 * kEpiWarps) {
                    const int rowi = w / 28, xi = w - rowi * 28;
                    const int oy = rowi >> 1, pyy = rowi & 1, ox = xi >> 1, pxx = xi & 1;
                    const int ggy = tc.gy0 + oy, ggx = tc.gx0 + ox;
                    if (ox >= p.tsx || ggy >= p.Hg || ggx >= p.Wg) continue;
                    const int j0 = (pyy * 2 + pxx) * 3;
                    float a0 = 0.f, a1 = 0.f, a2 = 0.f;
#pragma unroll
                    for (int t9 = 0; t9 < 9; ++t9) {
                        const int dy = t9 / 3 - 1, dx = t9 % 3 - 1;
                        const int ar = (oy + 1 + dy) * 16 + (ox + 1 + dx);        // A-tile pixel
                        const uint32_t a = gp + (uint32_t)((t9 * 128 + ar) * 48 + j0 * 4);
                        a0 += ldsf(a); a1 += ldsf(a + 4); a2 += ldsf(a + 8);
                    }
                    const int ry = 2 * ggy + pyy - p.crop_top, rx = 2 * ggx + pxx - p.crop_left;
                    if (ry < 0 || ry >= p.crop_H || rx < 0 || rx >= p.crop_W) continue;
                    const float c3[3] = {a0, a1, a2};
                    const size_t o = ((size_t)tc.b * p.crop_H + ry) * p.crop_W + rx;
#pragma unroll
                    for (int ch = 0; ch < 3; ++ch) {
                        const float xv = fminf(fmaxf(c3[ch] + s_bias[ch], 0.0f), 1.0f);
                        if (p.out_f32) p.out_f32[((size_t)tc.b * 3 + ch) * p.crop_H * p.crop_W + (size_t)ry * p.crop_W + rx] = xv;
                        if (p.out_u8) p.out_u8[o * 3 + ch] = (uint8_t)roundf(xv * 255.0f);
                    }
                }
                // P is reused by the next tile: everyone done reading
                named_bar_sync(3, 32 * kEpiWarps);
            } else if (p.pack4) {
                // packed g_s L4: channel group g takes sub-pixel phase g (columns 4g .. 4g+2), so
                // all 16 epilogue warps share the 12 outputs of each grid pixel
                float v[16];
                __syncwarp();
                tmem_ld16(taddr, v);
                float c3[3] = {v[0], v[1], v[2]};
#pragma unroll
                for (int ph = 1; ph < 4; ++ph)
                    if (g == ph) { c3[0] = v[4 * ph]; c3[1] = v[4 * ph + 1]; c3[2] = v[4 * ph + 2]; }
                const int ry = 2 * gy + (g >> 1) - p.crop_top, rx = 2 * gx + (g & 1) - p.crop_left;
                if (valid && ry >= 0 && ry < p.crop_H && rx >= 0 && rx < p.crop_W) {
                    const size_t o = ((size_t)tc.b * p.crop_H + ry) * p.crop_W + rx;
#pragma unroll
                    for (int ch = 0; ch < 3; ++ch) {
                        const float xv = fminf(fmaxf(c3[ch] + s_bias[ch], 0.0f), 1.0f);
                        if (p.out_f32) p.out_f32[((size_t)tc.b * 3 + ch) * p.crop_H * p.crop_W + (size_t)ry * p.crop_W + rx] = xv;
                        if (p.out_u8) p.out_u8[o * 3 + ch] = (uint8_t)roundf(xv * 255.0f);
                    }
                }
            } else {
                const int ncol16 = (p.BN + 15) / 16;
                for (int c = g; c < ncol16; c += kEpiGroups) {
                    float v[16];
                    __syncwarp();
                    tmem_ld16(taddr + c * 16, v);
                    const int cb = co0 + c * 16;
                    if (cb >= p.Cout) continue;                       // warp-uniform
                    const int nj = p.pack4 ? 16 : min(16, p.Cout - cb);
                    if (p.pack4) {
#pragma unroll
                        for (int j = 0; j < 16; ++j) v[j] += s_bias[j & 3];
                    } else if (p.ep != EP_PARTIAL) {
#pragma unroll
                        for (int i4 = 0; i4 < 4; ++i4) {
                            const float4 bb = lds4(s_bias + cb + 4 * i4);
                            v[4 * i4 + 0] += bb.x; v[4 * i4 + 1] += bb.y; v[4 * i4 + 2] += bb.z; v[4 * i4 + 3] += bb.w;
                        }
                    }
                    switch (p.ep) {
                    case EP_PARTIAL: {
                        if (valid) {
                            float4* dst = reinterpret_cast<float4*>(
                                p.part + ((((size_t)tc.split * p.batch + tc.b) * p.Hout + oy) * p.Wout + ox) * p.Cout + cb);
                            dst[0] = make_float4(v[0], v[1], v[2], v[3]);          // raw accumulator (no bias)
                            dst[1] = make_float4(v[4], v[5], v[6], v[7]);
                            dst[2] = make_float4(v[8], v[9], v[10], v[11]);
                            dst[3] = make_float4(v[12], v[13], v[14], v[15]);
                        }
                        break;
                    }
                    case EP_F32: {
                        if (valid) {
#pragma unroll
                            for (int j = 0; j < 16; ++j)
                                if (j < nj) p.out_f32[chw0 + (size_t)(cb + j) * HWo] = v[j];
                        }
                        break;
                    }
                    case EP_RELU: {
#pragma unroll
                        for (int j = 0; j < 16; ++j) v[j] = fmaxf(v[j], 0.0f);
                        if (valid && p.out_f32) {
#pragma unroll
                            for (int j = 0; j < 16; ++j)
                                if (j < nj) p.out_f32[chw0 + (size_t)(cb + j) * HWo] = v[j];
                        }
                        emit16(v, cb);
                        break;
                    }
                    case EP_YQUANT:
                    case EP_ZQUANT: {
                        int8_t* sym = reinterpret_cast<int8_t*>(p.out_sym);
                        float av[16];
                        int vsat = 0;
#pragma unroll
                        for (int j = 0; j < 16; ++j) {
                            const float m = s_mu[cb + j];
                            const int s = round_clamp(v[j] - m, p.L, vsat);
                            if (valid && j < nj) sym[chw0 + (size_t)(cb + j) * HWo] = (int8_t)s;
                            av[j] = (p.ep == EP_YQUANT) ? fabsf(v[j]) : (float)s + m;
                        }
                        if (valid) sat += vsat;
                        if (valid && p.out_f32) {
#pragma unroll
                            for (int j = 0; j < 16; ++j)
                                if (j < nj) p.out_f32[chw0 + (size_t)(cb + j) * HWo] = v[j];
                        }
                        if (p.out_act && (p.ep == EP_ZQUANT || p.abs_out)) emit16(av, cb);
                        break;
                    }
                    case EP_SIGMA: {
                        if (!valid) break;
                        uint8_t* idx = reinterpret_cast<uint8_t*>(p.out_sym);
                        const uint32_t tab = smem_u32(s_tab);
                        if (p.out_f32) {
#pragma unroll
                            for (int j = 0; j < 16; ++j)
                                if (j < nj) p.out_f32[chw0 + (size_t)(cb + j) * HWo] = fmaxf(v[j], 0.0f);
                        }
                        // sigma' = max(relu(x), 0.11); index = #{j in [0, 62] : table_j < sigma'}
                        // (sigma_index.cuh, the function lic_test_sigma_to_index checks exactly)
                        const auto ltab = [&](int i) { return ldsf(tab + 4u * (uint32_t)i); };
#pragma unroll
                        for (int j = 0; j < 16; ++j) {
                            const int lo = sigma_to_index(fmaxf(v[j], 0.0f), ltab);
                            if (j < nj) idx[chw0 + (size_t)(cb + j) * HWo] = (uint8_t)lo;
                        }
                        break;
                    }
                    case EP_FINAL: {
                        if (!valid) break;
#pragma unroll
                        for (int j = 0; j < 16; ++j) {
                            if (j >= nj) continue;
                            // packed phases: column j -> sub-pixel (j>>2) of grid pixel (gy, gx), channel j&3
                            const int ch = p.pack4 ? (j & 3) : cb + j;
                            if (p.pack4 && ch >= 3) continue;
                            const int yy = p.pack4 ? 2 * gy + ((j >> 3) & 1) : oy;
                            const int xx = p.pack4 ? 2 * gx + ((j >> 2) & 1) : ox;
                            const int ry = yy - p.crop_top, rx = xx - p.crop_left;
                            if (ry < 0 || ry >= p.crop_H || rx < 0 || rx >= p.crop_W) continue;
                            const float xv = fminf(fmaxf(v[j], 0.0f), 1.0f);
                            if (p.out_f32)
                                p.out_f32[(((size_t)tc.b * 3 + ch) * p.crop_H + ry) * p.crop_W + rx] = xv;
                            if (p.out_u8)
                                p.out_u8[(((size_t)tc.b * p.crop_H + ry) * p.crop_W + rx) * 3 + ch] =
                                    (uint8_t)roundf(xv * 255.0f);
                        }
                        break;
                    }
                    default: break;
                    }
                }
            }
            if (!released) {
                tc_fence_before();
                __syncwarp();
                if (lane == 0) {
                    if constexpr (CG == 2) mbar_arrive_cluster(lbar(&tempty_bar[buf]));
                    else mbar_arrive(&tempty_bar[buf]);
                }
            }
            if (threadIdx.x == 128) LIC_TRACE(it, T_EPI_END);
        }
        if (defer) flush_deferred();
        if (p.tma_out && lane == 0 && (g == 0 || p.wst_ch)) bulk_wait0();
        if (p.sat_count) {
            for (int o = 16; o > 0; o >>= 1) sat += __shfl_xor_sync(0xffffffffu, sat, o);
            if (lane == 0 && sat) atomicAdd(p.sat_count, (unsigned long long)sat);
        }
        if (p.range_count) {
            for (int o = 16; o > 0; o >>= 1) ovf += __shfl_xor_sync(0xffffffffu, ovf, o);
            if (lane == 0 && ovf) atomicAdd(p.range_count, (unsigned long long)ovf);
        }
    }

    tc_fence_before();
    // CG = 2: the leader's MMAs read the peer's smem and write its TMEM -- nobody leaves early
    if constexpr (CG == 2) cluster_sync_all(); else __syncthreads();
    if (warp == 2) {
        tc_fence_after();
        if constexpr (CG == 2) tmem_dealloc_cg2(tmem_base, (uint32_t)p.tmem_cols);
        else tmem_dealloc(tmem_base, (uint32_t)p.tmem_cols);
    }
}

template <int GC, int CG, bool L1>
static cudaError_t launch_t(const CUtensorMap& mapA, const CUtensorMap& mapB, const CUtensorMap& mapG,
                            const CUtensorMap& mapOH, const CUtensorMap& mapOL, const CUtensorMap& mapO2,
                            const CUtensorMap& mapO3, const ConvParams& p, int grid, cudaStream_t stream) {
    static bool attr_set = false;
    if (!attr_set) {
        cudaError_t e = cudaFuncSetAttribute(conv_umma_kernel<GC, CG, L1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             227 * 1024);
        if (e != cudaSuccess) return e;
        attr_set = true;
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = p.smem_bytes;
    cfg.stream = stream;
    cudaLaunchAttribute attr[2];
    int na = 0;
    if constexpr (CG == 2) {
        attr[na].id = cudaLaunchAttributeClusterDimension;
        attr[na].val.clusterDim.x = 2;
        attr[na].val.clusterDim.y = 1;
        attr[na].val.clusterDim.z = 1;
        ++na;
    }
    if (p.pdl) {
        attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[na].val.programmaticStreamSerializationAllowed = 1;
        ++na;
    }
    cfg.attrs = attr;
    cfg.numAttrs = na;
    return cudaLaunchKernelEx(&cfg, conv_umma_kernel<GC, CG, L1>, mapA, mapB, mapG, mapOH, mapOL, mapO2, mapO3, p);
}

cudaError_t launch_conv_umma(const CUtensorMap& mapA, const CUtensorMap& mapB, const CUtensorMap& mapG,
                             const CUtensorMap& mapOH, const CUtensorMap& mapOL, const CUtensorMap& mapO2,
                             const CUtensorMap& mapO3, const ConvParams& p, int grid, cudaStream_t stream) {
    const bool gdn = (p.ep == EP_GDN || p.ep == EP_IGDN);
#define LIC_LAUNCH(G, C, L) launch_t<G, C, L>(mapA, mapB, mapG, mapOH, mapOL, mapO2, mapO3, p, grid, stream)
    if (!gdn) return p.fuse_l1 ? cudaErrorInvalidValue : (p.cg == 2 ? LIC_LAUNCH(0, 2, false) : LIC_LAUNCH(0, 1, false));
    // GDN channel counts of the configs: N = 128, 192
    if (p.BN != 128 && p.BN != 192) return cudaErrorInvalidValue;
    if (p.cg == 2) {
        if (p.BN == 128) return p.fuse_l1 ? LIC_LAUNCH(2, 2, true) : LIC_LAUNCH(2, 2, false);
        return p.fuse_l1 ? LIC_LAUNCH(3, 2, true) : LIC_LAUNCH(3, 2, false);
    }
    if (p.BN == 128) return p.fuse_l1 ? LIC_LAUNCH(2, 1, true) : LIC_LAUNCH(2, 1, false);
    return p.fuse_l1 ? LIC_LAUNCH(3, 1, true) : LIC_LAUNCH(3, 1, false);
#undef LIC_LAUNCH
}

}  // namespace lic
