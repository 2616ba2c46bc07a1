// codec.cu -- the lic_codec runtime behind include/lic.h.
//
//  * parses + validates the LICW container and repacks the
//    weights into the GEMM engine's layout (fp16 W[tap][co][ci]);
//  * plans every transform layer once per (geometry, max_batch): GEMM grid, tile shape,
//    tap lists (conv / sub-pixel deconv phases), pipeline depth, TMEM budget, TMA maps;
//  * owns all device memory, allocated once in lic_open, freed in lic_close;
//  * owns a pinned, device-mapped host buffer pool (PAPER.md:84 zero-copy, :105 pooling);
//  * runs encode, hyper_indexes (decoder GPU1, :76) and decode (GPU2).
#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <set>
#include <string>
#include <vector>

#include "../../include/lic.h"
#include "internal.h"
#include "layer.h"

namespace lic {
cudaError_t launch_conv_umma(const CUtensorMap&, const CUtensorMap&, const CUtensorMap&, const CUtensorMap&,
                             const CUtensorMap&, const CUtensorMap&, const CUtensorMap&, const ConvParams&, int,
                             cudaStream_t);
cudaError_t launch_split_reduce(const float* part, int S, int B, int H, int W, int C, const float* bias,
                                const float* mu, int ep, int L, __half* out_act, size_t act_plane, int split,
                                int8_t* out_sym, float* out_f32, unsigned long long* sat_count,
                                unsigned long long* range_count, cudaStream_t st);
cudaError_t launch_sym_ingest(const int8_t*, const float*, int, int, int, int, __half*, size_t, int, cudaStream_t);
cudaError_t launch_pack_chw(const float*, int, int, int, int, __half*, size_t, int, cudaStream_t);
cudaError_t launch_sigma_index(const float*, size_t, const float*, uint8_t*, cudaStream_t);
}  // namespace lic

using namespace lic;

// ------------------------------------------------------------------ tensor-map encoder
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn get_encode_fn() {
    static EncodeTiledFn fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = (EncodeTiledFn)p;
    }
    return fn;
}

// TMA box semantics for strided traversal: boxDim counts elements of the *unstrided*
// footprint; the unit loads ceil(boxDim / elementStride) of them (CUDA driver API,
// cuTensorMapEncodeTiled "elementStrides").
#ifndef LIC_TMA_BOX_SCALED
#define LIC_TMA_BOX_SCALED 1
#endif

// ------------------------------------------------------------------ LICW format
namespace {

enum Role { R_CONV, R_DECONV, R_BIAS, R_BETA, R_GAMMA, R_PARAM };
struct BlockSpec { int tag; std::string name; Role role; std::vector<int> shape; bool hyper_only; };

std::vector<BlockSpec> licw_blocks(int N, int M) {
    std::vector<BlockSpec> b;
    int tag = 0;
    auto add = [&](const std::string& n, Role r, std::vector<int> s, bool h) { b.push_back({++tag, n, r, s, h}); };
    for (int i = 1; i <= 3; ++i) {
        int cin = i == 1 ? 3 : N;
        add("ga" + std::to_string(i) + ".w", R_CONV, {N, cin, 5, 5}, false);
        add("ga" + std::to_string(i) + ".b", R_BIAS, {N}, false);
        add("ga" + std::to_string(i) + ".beta", R_BETA, {N}, false);
        add("ga" + std::to_string(i) + ".gamma", R_GAMMA, {N, N}, false);
    }
    add("ga4.w", R_CONV, {M, N, 5, 5}, false);
    add("ga4.b", R_BIAS, {M}, false);
    for (int i = 1; i <= 3; ++i) {
        int cin = i == 1 ? M : N;
        add("gs" + std::to_string(i) + ".w", R_DECONV, {N, cin, 5, 5}, false);
        add("gs" + std::to_string(i) + ".b", R_BIAS, {N}, false);
        add("gs" + std::to_string(i) + ".beta", R_BETA, {N}, false);
        add("gs" + std::to_string(i) + ".gamma", R_GAMMA, {N, N}, false);
    }
    add("gs4.w", R_DECONV, {3, N, 5, 5}, false);
    add("gs4.b", R_BIAS, {3}, false);
    add("ha1.w", R_CONV, {N, M, 3, 3}, true);
    add("ha1.b", R_BIAS, {N}, true);
    add("ha2.w", R_CONV, {N, N, 5, 5}, true);
    add("ha2.b", R_BIAS, {N}, true);
    add("ha3.w", R_CONV, {N, N, 5, 5}, true);
    add("ha3.b", R_BIAS, {N}, true);
    add("hs1.w", R_DECONV, {N, N, 5, 5}, true);
    add("hs1.b", R_BIAS, {N}, true);
    add("hs2.w", R_DECONV, {N, N, 5, 5}, true);
    add("hs2.b", R_BIAS, {N}, true);
    add("hs3.w", R_CONV, {M, N, 3, 3}, true);
    add("hs3.b", R_BIAS, {M}, true);
    add("mu_y", R_PARAM, {M}, false);
    add("sigma_y", R_PARAM, {M}, false);
    add("mu_z", R_PARAM, {N}, true);
    add("sigma_z", R_PARAM, {N}, true);
    add("scale_table", R_PARAM, {64}, false);
    return b;
}

template <typename T>
T rd(const uint8_t* p) { T v; std::memcpy(&v, p, sizeof(T)); return v; }  // little-endian host

}  // namespace

// ------------------------------------------------------------------ codec state
enum LayerId { GA1 = 0, GA2, GA3, GA4, GS1, GS2, GS3, GS4, HA1, HA2, HA3, HS1, HS2, HS3, NLAYER };
static const char* kLayerW[NLAYER] = {"ga1", "ga2", "ga3", "ga4", "gs1", "gs2", "gs3", "gs4",
                                      "ha1", "ha2", "ha3", "hs1", "hs2", "hs3"};

struct Layer {
    bool present = false;
    bool deconv = false;
    int k = 5, s = 2, p = 2;
    int Cin = 0, Cin_eff = 0, Cout = 0;
    int Hin = 0, Win = 0, Hout = 0, Wout = 0;
    EpKind ep = EP_F32;
    __half* w = nullptr;      // [ntaps_w][Cout_pad][Cin_eff]
    float* bias = nullptr;
    float* beta = nullptr;
    __half* gamma = nullptr;  // [Cout][Cout]
    __half* in_buf = nullptr;
    size_t in_plane = 0;
    __half* out_buf = nullptr;
    size_t out_plane = 0;
    char in_id = 0, out_id = 0;   // workspace buffer ('A', 'B', 'Y', 'Z'; 0 = none) -- re-bound by lic_bind_workspace
    bool y_bounded = false;   // forward GDN / 1DN whose output provably stays in fp16 range (no guard)
    ConvParams prm{};
    CUtensorMap mapA{}, mapB{}, mapG{}, mapOH{}, mapOL{}, mapO2{}, mapO3{};
};

struct lic_codec {
    int device = 0, num_sms = 148;
    int kind = 0, act = 0, N = 0, M = 0, L = 32;
    int H = 0, W = 0, Hp = 0, Wp = 0, top = 0, left = 0;
    int max_batch = 1, split = 2;
    cudaStream_t stream = nullptr;
    std::string err;
    bool sticky = false;
    Layer layers[NLAYER];
    // device buffers
    __half *bufA = nullptr, *bufB = nullptr, *bufY = nullptr, *bufZ = nullptr;
    size_t planeA = 0, planeY = 0, planeZ = 0;
    float *mu_y = nullptr, *mu_z = nullptr, *table = nullptr;
    unsigned long long* d_sat = nullptr;
    unsigned long long* d_range = nullptr;   // activations saturated to the fp16 range (R16d)
    void* d_frames = nullptr;           // staging for host frames (f32 CHW size)
    int8_t* d_ysym = nullptr;
    uint8_t* d_yidx = nullptr;
    int8_t* d_zsym = nullptr;
    float* d_part = nullptr;                 // split-K partial sums (workspace)
    float* d_dbg = nullptr;             // test-layer / debug scratch
    float* d_dbg_in = nullptr;          // test-layer input copy for the fused g_a L1
    size_t dbg_elems = 0;
    float *dbg_y = nullptr, *dbg_z = nullptr, *dbg_s = nullptr;
    int debug = 0;
    int zero_copy = 0;
    std::vector<uint8_t> licw;     // the weights container, for lic_internal_clone
    int precision = 0;
    int halo_enabled = 1;          // LIC_NO_HALO=1 in the environment disables halo mode
    int tma_out_enabled = 1;       // LIC_TMA_OUT=0 disables the TMA-store epilogue
    int cg_enabled = 1;            // LIC_CG=1 forces one CTA per tile (no cta_group::2 pairs)
    int gs4_bn = 32;               // packed g_s L4 N tile (env LIC_GS4_BN=16|32)
    int pdl_enabled = 1;           // programmatic dependent launch of the GEMM engine (env LIC_PDL=0 disables)
    int small_bn = 0;              // N tile of the h_a / h_s layers (env LIC_SMALL_BN=64|96|128; 0 = whole Cout: measured no gain)
    int hs3_split_n = 1;           // h_s L3 with Cout 192 as two 96-channel N tiles (env LIC_HS3_SPLITN=0: off)
    int s2halo_enabled = 1;        // 5x5/s2 convs in parity-sub-grid halo mode (env LIC_S2HALO=0: per-tap tiles)
    int a_hi_only_enabled = 1;     // g_s L1 skips the zero lo plane of the integer y-hat (env LIC_YHAT_HI=0: off)
    int raw_tma_enabled = 1;       // u8 frames: raw patches by TMA (env LIC_RAW_TMA=0: cp.async)
    int ksplit_enabled = 1;        // split-K for the few-tile h layers (env LIC_KSPLIT=0: off, =2/3/4: at most that many slices)
    int ksplit_force = 0;
    int g2_slot16 = 1;             // two-group epilogue also with 32 KB of staging (16-channel rounds; env LIC_G2_SLOT16=0: off)
    int g2_192 = 1;                // two-group epilogue also for BN = 192 (chunked norm; env LIC_G2_192=0: off)
    int mma_spin = 0;              // g2 halo layers: MMA warp spins on operand barriers (env LIC_MMA_SPIN=1)
    int l1_stage_split = 1;        // u8 frames: hi-only A stages, twice as many (env LIC_L1_STAGES=0: off)
    int g2_enabled = 2;            // two-group GDN epilogue: 1 g_a L1 only, 2 every BN = 128 GDN layer (env LIC_G2)
    int l1_int_enabled = 1;        // u8 frames: integer samples into g_a L1, one MMA pass (env LIC_L1_INT=0: off)
    int l1_conv_enabled = 1;       // ... converted arithmetically, 8 per item, no LUT (env LIC_L1_CONV=0: LUT)
    int gs4_gather = 1;            // g_s L4 in gather mode (offsets in N; env LIC_GS4_GATHER=0: packed-phase halo mode)
    int wres_enabled = 1;          // env LIC_NO_WRES=1 streams the g_s L4 weights
    int wstage_enabled = 1;        // per-warp output staging in the GDN epilogue (env LIC_WSTAGE=0: quadrant blocks)
    int no_guard_enabled = 1;      // skip the range guard of provably bounded GDN outputs (env LIC_NO_GUARD=0: keep it)
    int gs1_hi_plan = 1;           // hyperprior g_s L1: hi-only halo ring, deeper weight ring (env LIC_GS1_HI=0: off)
    int g2_db16 = 0;               // two-group epilogue: double-buffered 16-channel staging (env LIC_G2_DB16=1 all, 2 g_a L1)
    int l1_rows_enabled = 1;       // u8 frames: row-halo g_a L1 (layer.h l1_rows; env LIC_L1_ROWS=0: im2col tiles)
    Layer l1r;                     // g_a L1 planned in row-halo mode (tile 8 x 16; shares GA1's weights and buffers)
    bool l1r_ok = false;
    Layer gs1h;                    // g_s L1 planned for a hi-only input (hyperprior decode; shares GS1's weights and buffers)
    bool gs1h_ok = false;
    std::vector<float> h_sigma_y, h_sigma_z, h_table, h_mu_y, h_mu_z;
    std::vector<uint32_t> cdf_fact, cdf_z, cdf_gauss;
    std::vector<void*> allocs;          // device allocations to free
    void* ws_own = nullptr;             // library-allocated workspace (nullptr once the caller binds one)
    void* ws_user = nullptr;            // caller-owned workspace (lic_bind_workspace)
    size_t ws_bytes = 0;
    int open_batch = 1;                 // max_batch given to lic_open (a bound workspace may lower max_batch)
    float* d_test = nullptr;            // test-only scratch (lic_test_sigma_to_index), allocated on first use
    uint8_t* d_test_idx = nullptr;
    // pinned pool
    std::mutex pool_mu;
    std::map<size_t, std::vector<void*>> free_lists;
    std::map<void*, size_t> owned;
    uint64_t pool_allocs = 0, pool_reuses = 0;
    // measurement
    uint64_t launches = 0;
    int profiling = 0;
    uint32_t prof_mask = 0;        // layers whose launches are bracketed by events
    int trace_layer = -1;
    unsigned long long* d_trace = nullptr;   // 256 tiles x 8 events
    std::vector<cudaEvent_t> ev;            // [2 * kProfSlots]
    std::vector<int> ev_layer;              // layer of each recorded pair
    int ev_used = 0;
    double prof_ms[NLAYER] = {0};
    uint64_t prof_n[NLAYER] = {0};
};
static constexpr int kProfSlots = 2048;

static void prof_flush(lic_codec* c) {
    if (!c->ev_used) return;
    cudaEventSynchronize(c->ev[2 * (c->ev_used - 1) + 1]);
    for (int i = 0; i < c->ev_used; ++i) {
        float ms = 0;
        cudaEventElapsedTime(&ms, c->ev[2 * i], c->ev[2 * i + 1]);
        c->prof_ms[c->ev_layer[i]] += ms;
        c->prof_n[c->ev_layer[i]] += 1;
    }
    c->ev_used = 0;
}

static lic_status fail(lic_codec* c, lic_status st, const char* fmt, ...) {
    if (c) {
        char buf[512];
        va_list ap;
        va_start(ap, fmt);
        vsnprintf(buf, sizeof buf, fmt, ap);
        va_end(ap);
        c->err = buf;
        if (st == LIC_ECUDA) c->sticky = true;
    }
    return st;
}

#define CK(call)                                                                               \
    do {                                                                                       \
        cudaError_t e_ = (call);                                                               \
        if (e_ != cudaSuccess) return fail(c, LIC_ECUDA, "%s: %s", #call, cudaGetErrorString(e_)); \
    } while (0)

template <typename T>
static lic_status dalloc(lic_codec* c, T** p, size_t bytes) {
    void* q = nullptr;
    if (cudaMalloc(&q, bytes ? bytes : 16) != cudaSuccess) {
        cudaGetLastError();
        return fail(c, LIC_ENOMEM, "cudaMalloc(%zu) failed", bytes);
    }
    c->allocs.push_back(q);
    *p = (T*)q;
    return LIC_OK;
}

// ------------------------------------------------------------------ planning helpers
// plane_elems: distance between the hi and lo planes of the buffer (its full plane size,
// which exceeds B*H*W*C when a large buffer is reused by a smaller layer)
static bool encode_act_map(CUtensorMap* m, const __half* base, int C, int W, int H, int B, int planes,
                           size_t plane_elems, int box_w, int box_h, int es) {
    EncodeTiledFn enc = get_encode_fn();
    if (!enc) return false;
    cuuint64_t dims[5] = {(cuuint64_t)C, (cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)B, (cuuint64_t)planes};
    cuuint64_t str[4] = {(cuuint64_t)C * 2, (cuuint64_t)W * C * 2, (cuuint64_t)H * W * C * 2,
                         (cuuint64_t)plane_elems * 2};
#if LIC_TMA_BOX_SCALED
    cuuint32_t box[5] = {64, (cuuint32_t)(box_w * es), (cuuint32_t)(box_h * es), 1, 1};
#else
    cuuint32_t box[5] = {64, (cuuint32_t)box_w, (cuuint32_t)box_h, 1, 1};
#endif
    cuuint32_t es5[5] = {1, (cuuint32_t)es, (cuuint32_t)es, 1, 1};
    return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 5, (void*)base, dims, str, box, es5, CU_TENSOR_MAP_INTERLEAVE_NONE,
               CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// the u8 HWC frames as a 3-D byte tensor (3W, H, B), box = one fused-L1 raw patch (128 B x 19 rows)
// (row-halo g_a L1: 80 B x 35 rows)
static bool encode_u8_frame_map(CUtensorMap* m, const void* base, int W, int H, int B, bool rows = false) {
    EncodeTiledFn enc = get_encode_fn();
    if (!enc) return false;
    cuuint64_t dims[3] = {(cuuint64_t)W * 3, (cuuint64_t)H, (cuuint64_t)B};
    cuuint64_t str[2] = {(cuuint64_t)W * 3, (cuuint64_t)W * 3 * H};
    cuuint32_t box[3] = {rows ? 80u : 128u, rows ? 35u : 19u, 1};
    cuuint32_t es[3] = {1, 1, 1};
    return enc(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<void*>(base), dims, str, box, es,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

static bool encode_w_map(CUtensorMap* m, const __half* base, int K, int rows, int depth, int box_rows) {
    EncodeTiledFn enc = get_encode_fn();
    if (!enc) return false;
    cuuint64_t dims[3] = {(cuuint64_t)K, (cuuint64_t)rows, (cuuint64_t)depth};
    cuuint64_t str[2] = {(cuuint64_t)K * 2, (cuuint64_t)rows * K * 2};
    cuuint32_t box[3] = {64, (cuuint32_t)box_rows, 1};
    cuuint32_t es[3] = {1, 1, 1};
    return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 3, (void*)base, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
               CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// TMA-store maps of an NHWC fp16 plane, box = bc channels x one epilogue quadrant's 32 px:
// bc = 64 (128-byte rows, 128B swizzle: quadrant blocks) or 32 / 16 (64B / 32B swizzle:
// per-warp staging rounds)
static CUtensorMapSwizzle swz_for(int bc) {
    return bc == 64 ? CU_TENSOR_MAP_SWIZZLE_128B : bc == 32 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_32B;
}
static bool encode_out_conv_map(CUtensorMap* m, const __half* base, int C, int W, int H, int B, int bw, int bh,
                                int bc = 64) {
    EncodeTiledFn enc = get_encode_fn();
    if (!enc) return false;
    cuuint64_t dims[4] = {(cuuint64_t)C, (cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)B};
    cuuint64_t str[3] = {(cuuint64_t)C * 2, (cuuint64_t)W * C * 2, (cuuint64_t)H * W * C * 2};
    cuuint32_t box[4] = {(cuuint32_t)bc, (cuuint32_t)bw, (cuuint32_t)bh, 1};
    cuuint32_t es[4] = {1, 1, 1, 1};
    return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 4, (void*)base, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
               swz_for(bc), CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
// sub-pixel phase view of a stride-2 transposed conv output (NHWC, H = 2 Hin, W = 2 Win):
// dims (C, px, qx = x/2, py, qyb = b*Hin + y/2)
static bool encode_out_phase_map(CUtensorMap* m, const __half* base, int C, int W, int H, int B, int bw, int bh,
                                 int bc = 64) {
    EncodeTiledFn enc = get_encode_fn();
    if (!enc) return false;
    cuuint64_t dims[5] = {(cuuint64_t)C, 2, (cuuint64_t)(W / 2), 2, (cuuint64_t)B * (H / 2)};
    cuuint64_t str[4] = {(cuuint64_t)C * 2, (cuuint64_t)2 * C * 2, (cuuint64_t)W * C * 2, (cuuint64_t)2 * W * C * 2};
    cuuint32_t box[5] = {(cuuint32_t)bc, 1, (cuuint32_t)bw, 1, (cuuint32_t)bh};
    cuuint32_t es[5] = {1, 1, 1, 1, 1};
    return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 5, (void*)base, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
               swz_for(bc), CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// Per-warp staging (P.wst_ch): one bulk tensor store writes both planes (hi, lo) of a warp's
// 32 px x bc channels.  conv: (C, W, H, B, plane); stride-2 transposed conv: one map per
// sub-pixel phase (py, px), based at output pixel (py, px): (C, W/2 [2C], B*H/2 [2WC], plane)
static bool encode_out_conv_map_pl(CUtensorMap* m, const __half* base, int C, int W, int H, int B, size_t plane,
                                   int planes, int bw, int bh, int bc) {
    EncodeTiledFn enc = get_encode_fn();
    if (!enc) return false;
    cuuint64_t dims[5] = {(cuuint64_t)C, (cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)B, (cuuint64_t)planes};
    cuuint64_t str[4] = {(cuuint64_t)C * 2, (cuuint64_t)W * C * 2, (cuuint64_t)H * W * C * 2, (cuuint64_t)plane * 2};
    cuuint32_t box[5] = {(cuuint32_t)bc, (cuuint32_t)bw, (cuuint32_t)bh, 1, (cuuint32_t)planes};
    cuuint32_t es[5] = {1, 1, 1, 1, 1};
    return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 5, (void*)base, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
               swz_for(bc), CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
static bool encode_out_phase_map_pl(CUtensorMap* m, const __half* base, int C, int W, int H, int B, size_t plane,
                                    int planes, int ph, int bw, int bh, int bc) {
    EncodeTiledFn enc = get_encode_fn();
    if (!enc) return false;
    const __half* b0 = base + ((size_t)(ph >> 1) * W + (ph & 1)) * C;
    cuuint64_t dims[4] = {(cuuint64_t)C, (cuuint64_t)(W / 2), (cuuint64_t)B * (H / 2), (cuuint64_t)planes};
    cuuint64_t str[3] = {(cuuint64_t)2 * C * 2, (cuuint64_t)2 * W * C * 2, (cuuint64_t)plane * 2};
    cuuint32_t box[4] = {(cuuint32_t)bc, (cuuint32_t)bw, (cuuint32_t)bh, (cuuint32_t)planes};
    cuuint32_t es[4] = {1, 1, 1, 1};
    return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 4, (void*)b0, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
               swz_for(bc), CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// choose Wt x Ht = 128 minimising padded tiles over the grid
static void choose_tile(int Hg, int Wg, int* Wt, int* Ht) {
    static const int opts[5][2] = {{16, 8}, {32, 4}, {8, 16}, {64, 2}, {128, 1}};
    long best = -1;
    for (auto& o : opts) {
        long tiles = (long)((Wg + o[0] - 1) / o[0]) * ((Hg + o[1] - 1) / o[1]);
        if (best < 0 || tiles < best) { best = tiles; *Wt = o[0]; *Ht = o[1]; }
    }
}

// mbarrier area: full/empty[<= 8] + tfull/tempty[2] + norm + gamma + hfull/hempty[4] + xsq +
// wres (34 x 8 B) + the TMEM base slot
static constexpr uint32_t kBarBytes = 512;
constexpr int kKsplitMax = 4;                // split-K slices of the few-tile h layers (run_layer)
static constexpr int kGatherN = 144;     // g_s L4 gather mode: 9 input offsets x 16 packed outputs
static_assert(kBarBytes >= (2 * 8 + 2 * 2 + 2 + 2 * 4 + 2) * 8 + 4, "barrier area too small");

// q = (umulhi(n, m) + n) >> s == n / d for 0 <= n < 2^31 (round-up magic, d >= 1)
static void fast_div(int d, uint32_t* m, int* s) {
    int l = 0;
    while ((1ll << l) < d) ++l;
    *s = l;
    *m = (uint32_t)(((1ull << 32) * ((1ull << l) - (uint64_t)d)) / (uint64_t)d + 1);
}
static int ilog2_exact(int v) {
    for (int l = 0; l < 31; ++l) if ((1 << l) == v) return l;
    return -1;
}

static int pow2_cols(int n) {
    int c = 32;
    while (c < n) c <<= 1;
    return c;
}

// build the GEMM-side plan of one layer (everything except epilogue output pointers)
// layer id of a Layer (the row-halo g_a L1 plan counts as g_a L1)
static int lid_of(const lic_codec* c, const Layer& Ly) {
    if (&Ly == &c->gs1h) return GS1;
    return &Ly == &c->l1r ? (int)GA1 : (int)(&Ly - c->layers);
}

static lic_status plan_layer(lic_codec* c, Layer& Ly) {
    ConvParams& P = Ly.prm;
    const bool l1rows = &Ly == &c->l1r;
    std::memset(&P, 0, sizeof P);
    P.tps = 1;
    const bool gemm_l1 = (&Ly == &c->layers[GA1]) || l1rows;
    P.Cin = Ly.Cin_eff;
    P.kchunks = Ly.Cin_eff / 64;
    P.Cout = Ly.Cout;
    const bool gs4g = Ly.ep == EP_FINAL && Ly.deconv && c->gs4_gather;
    P.tsx = 0; P.tsy = 0;
    if (gs4g) { P.BN = kGatherN; P.n_ntiles = 1; }
    else if (Ly.ep == EP_FINAL && Ly.deconv) { P.BN = c->gs4_bn; P.n_ntiles = 1; }
    else if (Ly.Cout <= 256) { P.BN = (Ly.Cout + 15) / 16 * 16; P.n_ntiles = 1; }
    else { P.n_ntiles = (Ly.Cout + 255) / 256; P.BN = ((Ly.Cout + P.n_ntiles - 1) / P.n_ntiles + 15) / 16 * 16; }
    // h_a / h_s run on a few dozen pixel tiles (one per CTA pair, a serial load -> MMA ->
    // epilogue chain each): split their output channels into 64-wide N tiles so more CTAs work
    // and each CTA pipelines several tiles (env LIC_SMALL_BN=0 keeps one N tile)
    {
        const int lid = lid_of(c, Ly);
        const bool hyper_layer = lid >= HA1 && lid <= HS3;
        if (hyper_layer && c->small_bn && Ly.Cout % c->small_bn == 0 && Ly.Cout > c->small_bn &&
            Ly.ep != EP_GDN && Ly.ep != EP_IGDN) {
            P.BN = c->small_bn;
            P.n_ntiles = Ly.Cout / c->small_bn;
        } else if (lid == HS3 && !c->small_bn && c->hs3_split_n && Ly.Cout == 192) {
            // h_s L3 (sigma -> index, one 192-channel tile per CTA): two 96-channel N tiles, so a
            // CTA's second tile's MMAs overlap its first tile's epilogue (30 -> 28 us at C3)
            P.BN = 96;
            P.n_ntiles = 2;
        }
    }
    const bool gdn = (Ly.ep == EP_GDN || Ly.ep == EP_IGDN);
    if (gdn && (P.n_ntiles != 1 || P.BN != Ly.Cout || Ly.Cout % 64))
        return fail(c, LIC_EINVAL, "GDN layer needs Cout %% 64 == 0 and Cout <= 256");
    P.split = c->split;
    int ntap = 0;
    if (gemm_l1) {
        P.Hg = Ly.Hout; P.Wg = Ly.Wout; P.stride = 1; P.out_s = 1; P.nphase = 1;
        P.tap0[0] = 0; P.ntaps[0] = 1; P.tap_dy[0] = 0; P.tap_dx[0] = 0; P.tap_w[0] = 0;
        ntap = 1;
    } else if (!Ly.deconv && Ly.k == 5 && Ly.s == 2 && c->s2halo_enabled && c->halo_enabled) {
        // 5x5 / stride 2 / pad 2 conv as four stride-1 convolutions over the input's parity
        // sub-grids (py, px): tap (ky, kx) reads sub-grid (ky % 2, kx % 2) at offset
        // ((ky - py) / 2 - 1, (kx - px) / 2 - 1) in [-1, 1]^2 of the output pixel, so each
        // sub-grid contributes through a (Wt + 2) x (Ht + 2) halo (loaded with TMA element
        // stride 2) and its taps are shifted windows of it -- 4 halo loads per 64-channel chunk
        // instead of 25 tap tiles.  Groups g = py * 2 + px with 9 / 6 / 6 / 4 taps.
        P.Hg = Ly.Hout; P.Wg = Ly.Wout; P.stride = 2; P.out_s = 1; P.nphase = 1; P.sub4 = 1;
        for (int g = 0; g < 4; ++g) {
            const int py = g >> 1, px = g & 1;
            P.tap0[g] = ntap;
            for (int ky = py; ky < 5; ky += 2)
                for (int kx = px; kx < 5; kx += 2) {
                    P.tap_dy[ntap] = (ky - py) / 2 - 1; P.tap_dx[ntap] = (kx - px) / 2 - 1;
                    P.tap_w[ntap] = ky * 5 + kx; ++ntap;
                }
            P.ntaps[g] = ntap - P.tap0[g];
        }
    } else if (!Ly.deconv) {
        P.Hg = Ly.Hout; P.Wg = Ly.Wout; P.stride = Ly.s; P.out_s = 1; P.nphase = 1;
        P.tap0[0] = 0;
        for (int ky = 0; ky < Ly.k; ++ky)
            for (int kx = 0; kx < Ly.k; ++kx) {
                P.tap_dy[ntap] = ky - Ly.p; P.tap_dx[ntap] = kx - Ly.p; P.tap_w[ntap] = ky * Ly.k + kx; ++ntap;
            }
        P.ntaps[0] = ntap;
    } else if (gs4g) {
        // g_s L4 gather mode: one "tap" -- the 16 x 8 input tile itself, starting one pixel
        // up-left of the 14 x 6 output interior; B rows t*16 + phase*4 + co (9 offsets t)
        P.Hg = Ly.Hin; P.Wg = Ly.Win; P.stride = 1; P.out_s = 2; P.nphase = 1; P.gather = 1;
        P.tap0[0] = 0; P.ntaps[0] = 1; P.tap_dy[0] = -1; P.tap_dx[0] = -1; P.tap_w[0] = 0;
        ntap = 1;
    } else if (Ly.ep == EP_FINAL) {
        // g_s L4 (Cout = 3): all 4 sub-pixel phases packed into one N = 16 GEMM over the 9
        // input offsets (dy, dx) in {-1,0,1}^2 shared by the phases; B row (phase*4 + co)
        // holds W[co][.][ky][kx] with ky = py + 2 - 2dy, kx = px + 2 - 2dx (zero if outside).
        P.Hg = Ly.Hin; P.Wg = Ly.Win; P.stride = 1; P.out_s = 2; P.nphase = 1; P.pack4 = 1;
        P.tap0[0] = 0;
        for (int dy = -1; dy <= 1; ++dy)
            for (int dx = -1; dx <= 1; ++dx) {
                P.tap_dy[ntap] = dy; P.tap_dx[ntap] = dx; P.tap_w[ntap] = ntap; ++ntap;
            }
        P.ntaps[0] = ntap;
    } else {
        // stride-2 5x5 transposed conv, p = 2, output_padding 1: output (2qy+py, 2qx+px) takes
        // taps ky = py (mod 2) from input row qy + (py + 2 - ky)/2 (same for x).
        P.Hg = Ly.Hin; P.Wg = Ly.Win; P.stride = 1; P.out_s = 2; P.nphase = 4;
        for (int ph = 0; ph < 4; ++ph) {
            const int py = ph >> 1, px = ph & 1;
            P.tap0[ph] = ntap;
            for (int ky = py; ky < 5; ky += 2)
                for (int kx = px; kx < 5; kx += 2) {
                    P.tap_dy[ntap] = (py + 2 - ky) / 2; P.tap_dx[ntap] = (px + 2 - kx) / 2;
                    P.tap_w[ntap] = ky * 5 + kx; ++ntap;
                }
            P.ntaps[ph] = ntap - P.tap0[ph];
        }
    }
    // CTA pair (cta_group::2, M = 256) unless disabled (env LIC_CG=1); B / gamma split by rows
    // (N tiles >= 64 only: the packed N = 16 g_s L4 stays on one CTA per tile)
    P.cg = (c->cg_enabled && P.BN % 16 == 0 && P.BN >= 32 && !gs4g) ? 2 : 1;
    // shared memory plan: stage ring | halo ring (halo mode) | gamma (GDN) | mbarriers | constants
    const uint32_t a_bytes = 128 * 64 * 2, b_bytes = (uint32_t)(P.BN / P.cg) * 64 * 2;
    const uint32_t gamma_bytes = gdn ? (uint32_t)(P.BN / 64) * b_bytes : 0;
    // bias / beta / mu, scale table, halo tap offsets (+ GDN: per-pixel norm exponents, 128 x 4 B)
    const uint32_t par_bytes = (uint32_t)(3 * P.BN * P.n_ntiles + 64 + kMaxTaps) * 4 + (gdn ? 1024u : 0u);
    const uint32_t budget = 227u * 1024u;
    // TMA-store epilogue: 4 lane quadrants x 8 KB block slots (1 or 2 slots), when the layer writes an activation and the
    // pipeline keeps >= 3 stages with it (env LIC_TMA_OUT=0 disables)
    // (64-channel store blocks: N tiles that are not a multiple of 64 -- g_a L4 at M = 320, two
    // N tiles of 160 -- store directly)
    const bool has_act = Ly.out_buf != nullptr && Ly.ep != EP_SIGMA && Ly.ep != EP_FINAL && P.BN % 64 == 0;
    bool tma_out = has_act && c->tma_out_enabled;
    const uint32_t ostage_bytes = 16 * 2048;
    {
        const uint32_t fx = gamma_bytes + kBarBytes + par_bytes + 1024 + ostage_bytes;
        const uint32_t st_b = a_bytes * P.split + b_bytes;     // per-tap stage (non-halo)
        const bool stride1_ = !gemm_l1 && (Ly.deconv || (Ly.k == 3 && Ly.s == 1) || P.sub4);
        if (!stride1_ && fx + 3 * st_b > budget) tma_out = false;
    }
    const uint32_t fixed = gamma_bytes + kBarBytes + par_bytes + 1024 + (tma_out ? ostage_bytes : 0);
    // halo mode: every stride-1 layer whose taps stay inside a 3x3 neighbourhood
    const bool stride1 = !gemm_l1 && (Ly.deconv || (Ly.k == 3 && Ly.s == 1) || P.sub4);
    int halo_w = 10;                                                   // Wt + 2
    if (const char* e = std::getenv("LIC_HALO_W")) halo_w = std::max(10, std::min(32, atoi(e)));
    const uint32_t hpb = ((uint32_t)(halo_w * 18 * 128) + 1023) / 1024 * 1024;   // halo_w x (Ht+2) rows
    // the hyperprior's g_s L1 on the decode path reads a hi-only input (R16c): one plane per halo slot,
    // the freed shared memory goes to the weight ring (c->gs1h)
    const bool hi_only_plan = &Ly == &c->gs1h;
    const int hplanes = hi_only_plan ? 1 : P.split;
    P.halo_planes = hplanes;
    P.a_hi_only = hi_only_plan ? 1 : 0;
    if (l1rows) {
        // row-halo g_a L1 (u8 frames; layer.h l1_rows): stage = one 35 x 8-row halo (SW128 rows),
        // 3 stages when they fit; resident weights; 2 raw u8 patch slots (TMA, 80 B x 35 rows)
        P.fuse_l1 = 1;
        P.l1_rows = 1;
        P.halo = 0;
        P.halo_slots = 0;
        P.Wt = 8; P.Ht = 16;
        P.stage_bytes = 35u * 8u * 128u;
        const uint32_t wbytes = (uint32_t)P.kchunks * b_bytes, rawb = 2u * 2816u;
        P.stages = (fixed + 3 * P.stage_bytes + wbytes + rawb + 2048 + (tma_out ? ostage_bytes : 0) <= budget) ? 3 : 2;
        P.wres = 1;
        P.off_wres = P.stages * P.stage_bytes;
        P.off_patch = P.off_wres + wbytes;
        P.off_lut = P.off_patch;
        P.off_halo = 0;
        P.off_raw = (P.off_patch + 127) / 128 * 128;
        P.off_gamma = (P.off_raw + rawb + 1023) / 1024 * 1024;
    } else if (gemm_l1) {
        // fused g_a L1: stage s = A chunk s (hi, lo) built by warps 0/2/3; resident weights;
        // double-buffered fp32 input patch; k -> patch offset table + u8 LUT
        P.fuse_l1 = 1;
        P.halo = 0;
        P.halo_slots = 0;
        P.Wt = 16; P.Ht = 8;
        P.stage_bytes = a_bytes * P.split;
        P.stages = P.kchunks;
        P.wres = 1;
        P.off_wres = P.stages * P.stage_bytes;
        P.off_patch = P.off_wres + P.kchunks * b_bytes;
        const uint32_t patch_bytes = 2u * 19u * 112u * 2u;           // hi + lo planes
        P.off_lut = P.off_patch + 2 * patch_bytes;
        P.off_halo = 0;
        P.off_raw = (P.off_lut + 257 * 4 + 127) / 128 * 128;
        P.off_gamma = (P.off_raw + 2 * 19 * 128 + 1023) / 1024 * 1024;     // raw: 2 x 19 rows x 128 B
    } else if (gs4g) {
        P.halo = 0;
        P.halo_slots = 0;
        P.Wt = 16; P.Ht = 8;
        P.tsx = 14; P.tsy = 6;
        P.stage_bytes = a_bytes * P.split;
        P.stages = 3;
        P.wres = 1;
        P.off_wres = P.stages * P.stage_bytes;
        P.off_gp = P.off_wres + P.kchunks * b_bytes;
        P.off_halo = 0;
        P.off_gamma = (P.off_gp + 9u * 128u * 48u + 1023) / 1024 * 1024;
    } else if (stride1 && fixed + 2 * hplanes * hpb + 2 * b_bytes <= budget && c->halo_enabled) {
        P.halo = 1;
        P.Wt = 8; P.Ht = 16;
        P.halo_plane_bytes = hpb;
        P.halo_w = halo_w;
        // several taps per weight stage (one wait per 8 * tps MMAs; env LIC_TPS=1..4)
        // (measured per layer: 3 for the many-tile parity-halo convs of g_a, 2 elsewhere)
        {
            const int lid = lid_of(c, Ly);
            // (the hi-only g_s L1 plan too: a weight tile feeds only 4 MMAs there, 3 taps per wait
            // measured 6 % faster than 2)
            P.tps = ((P.sub4 && lid >= GA2 && lid <= GA4) || hi_only_plan) ? 3 : 2;
        }
        if (const char* e = std::getenv("LIC_TPS")) P.tps = std::max(1, std::min(kMaxTps, atoi(e)));
        P.stage_bytes = b_bytes * (uint32_t)P.tps;
        // halo ring depth: env LIC_HALO_SLOTS (2..4, default 2: a halo chunk is reused by all
        // its taps, while every tap needs a fresh weight tile, so smem goes to the weight ring)
        int slots = 2;
        if (const char* e = std::getenv("LIC_HALO_SLOTS")) slots = std::max(2, std::min(4, atoi(e)));
        while (slots > 2 && fixed + slots * hplanes * hpb + 3 * b_bytes > budget) --slots;
        P.halo_slots = slots;
        // small weight sets (packed g_s L4: 9 taps x 2 chunks x 2 KB) stay resident
        const uint32_t wtot = (uint32_t)P.ntaps[0] * P.kchunks * b_bytes;
        if (c->wres_enabled && P.nphase == 1 && fixed + slots * hplanes * hpb + wtot <= budget && wtot <= 64 * 1024) {
            P.wres = 1;
            P.stages = 1;
            P.stage_bytes = 0;
            P.off_wres = 0;
            P.off_halo = (wtot + 1023) / 1024 * 1024;
        } else {
            int stages = (int)((budget - fixed - slots * hplanes * hpb) / P.stage_bytes);
            // keep a double-buffered weight ring: wide N tiles (M = 320 models, BN = 192) drop to
            // fewer taps per stage rather than to a single stage (measured: -10% frames/s at 1 stage)
            while (stages < 2 && P.tps > 1) {
                --P.tps;
                P.stage_bytes = b_bytes * (uint32_t)P.tps;
                stages = (int)((budget - fixed - slots * hplanes * hpb) / P.stage_bytes);
            }
            P.stages = std::min(stages, 8);
            P.off_halo = P.stages * P.stage_bytes;
        }
        P.off_gamma = P.off_halo + slots * hplanes * hpb;
    } else {
        P.halo = 0;
        P.halo_slots = 0;
        choose_tile(P.Hg, P.Wg, &P.Wt, &P.Ht);
        P.stage_bytes = a_bytes * P.split + b_bytes;
        int stages = (int)((budget - fixed) / P.stage_bytes);
        stages = std::min(stages, 8);
        if (stages < 2) return fail(c, LIC_EINVAL, "layer does not fit shared memory");
        P.stages = stages;
        P.off_halo = 0;
        P.off_gamma = stages * P.stage_bytes;
    }
    if (P.sub4 && !P.halo) return fail(c, LIC_EINVAL, "parity-halo conv does not fit shared memory");
    for (int i = 0; i < kMaxTaps; ++i)
        P.tapoff[i] = P.halo ? (uint32_t)(((P.tap_dy[i] + 1) * P.halo_w + P.tap_dx[i] + 1) * 8) : 0u;
    if (!P.tsx) { P.tsx = P.Wt; P.tsy = P.Ht; }
    P.tiles_x = (P.Wg + P.tsx - 1) / P.tsx;
    P.tiles_y = (P.Hg + P.tsy - 1) / P.tsy;
    P.txs = (P.tiles_x + P.cg - 1) / P.cg;
    fast_div(P.n_ntiles, &P.fd_nt_m, &P.fd_nt_s);
    fast_div(P.txs, &P.fd_txs_m, &P.fd_txs_s);
    fast_div(P.tiles_y, &P.fd_ty_m, &P.fd_ty_s);
    P.wt_log2 = ilog2_exact(P.Wt);
    P.nph_log2 = ilog2_exact(P.nphase);
    if (P.wt_log2 < 0 || P.nph_log2 < 0) return fail(c, LIC_EINVAL, "tile width / phase count must be powers of two");
    P.off_bar = P.off_gamma + gamma_bytes;
    P.off_par = P.off_bar + kBarBytes;
    P.tma_out = tma_out ? 1 : 0;
    P.ostage_slots = 1;
    P.off_ostage = (P.off_par + par_bytes + 1023) / 1024 * 1024;
    P.smem_bytes = (tma_out ? P.off_ostage + ostage_bytes : P.off_par + par_bytes) + 1024;
    // double-buffered staging when it fits without losing pipeline depth below 3 (halo: 2) stages
    static const int ostage_max = [] {                     // env LIC_OSTAGE=1: single staging slot
        const char* e = std::getenv("LIC_OSTAGE");
        return (e && e[0] == '1') ? 1 : 2;
    }();
    if (ostage_max < 2) {
        // keep the smem for the operand rings
    } else if (tma_out && P.smem_bytes + ostage_bytes <= budget) {
        const bool keep = P.fuse_l1 || (P.halo ? (P.wres || P.stages >= 2) : P.stages >= 3);
        if (keep) { P.ostage_slots = 2; P.smem_bytes += ostage_bytes; }
    } else if (tma_out && P.halo && !P.wres && P.stage_bytes) {
        // trade weight stages (keeping >= 2) for the second staging slot
        const int drop = (int)((ostage_bytes + P.stage_bytes - 1) / P.stage_bytes);
        if (P.stages - drop >= 2) {
            const uint32_t sh = (uint32_t)drop * P.stage_bytes;
            P.stages -= drop;
            P.off_halo -= sh;
            P.off_gamma -= sh;
            P.off_bar -= sh;
            P.off_par -= sh;
            P.off_ostage = (P.off_par + par_bytes + 1023) / 1024 * 1024;
            P.ostage_slots = 2;
            P.smem_bytes = P.off_ostage + 2 * ostage_bytes + 1024;
        }
    }
    if (P.smem_bytes < 120 * 1024) P.smem_bytes = 120 * 1024;     // one CTA per SM (TMEM)
    if (P.smem_bytes > budget) return fail(c, LIC_EINVAL, "layer plan exceeds shared memory (%u)", P.smem_bytes);
    // two-group GDN epilogue (env LIC_G2: 0 off, 1 g_a L1 only, 2 every eligible GDN
    // layer): BN = 128, or BN = 192 with the norm in three 64-column chunks; needs 64 KB of
    // per-warp output staging (4 KB, 32-channel rounds)
    P.g2 = 0;
    if (gdn && (P.BN == 128 || (P.BN == 192 && c->g2_192)) && tma_out && c->wstage_enabled &&
        (P.ostage_slots == 2 || c->g2_slot16) && (gemm_l1 ? c->g2_enabled >= 1 : c->g2_enabled >= 2))
        P.g2 = 1;
    // TMEM plan: accumulator (+ GDN norm) per buffer, double-buffered when it fits (two-group
    // BN = 192: 192 + one 64-column norm chunk)
    int per = std::max(32, P.BN) + (gdn ? (P.g2 && P.BN == 192 ? 64 : P.BN) : 0);
    P.n_accbuf = (2 * per <= 512) ? 2 : 1;
    P.acc_stride = per;
    P.tmem_cols = pow2_cols(P.n_accbuf * per);
    if (P.g2 && P.n_accbuf != 2) P.g2 = 0;
    // per-warp staging of the GDN / IGDN epilogue when 64 KB of staging fit: rounds of 32 channels
    // (BN = 128: one round, one 4 KB slot per warp; two-group: one round per 32-channel sub-block)
    // or 16 (BN = 192 single group: three rounds, two 2 KB slots)
    P.wst_ch = 0;
    P.wst_slots = 0;
    if (gdn && tma_out && P.ostage_slots == 2 && c->wstage_enabled) {
        const int G = P.BN / 4;                                         // channels per epilogue warp
        P.wst_ch = (G % 32 == 0 || P.g2) ? 32 : 16;
        P.wst_slots = P.wst_ch == 32 ? 1 : 2;
        // two-group epilogue: 16-channel rounds in two alternating 2 KB slots per warp instead of one
        // 4 KB 32-channel slot (env LIC_G2_DB16=1 every such layer, 2 g_a L1 only; measured: no change)
        if (P.g2 && (c->g2_db16 == 1 || (c->g2_db16 == 2 && gemm_l1))) { P.wst_ch = 16; P.wst_slots = 2; }
    } else if (P.g2) {
        // two-group epilogue with 32 KB of staging: one 2 KB slot per warp, 16-channel rounds
        P.wst_ch = 16;
        P.wst_slots = 1;
    }
    P.mma_spin = (P.g2 && !gemm_l1 && c->mma_spin) ? 1 : 0;
    {
        // split-K candidates: the h layers with a handful of tiles (h_a L2, L3, h_s L1), whose
        // epilogue split_reduce_kernel implements (ReLU, z-quantise) and whose MMA loop is the
        // lean halo loop (the only one that iterates a K slice)
        const int lid = lid_of(c, Ly);
        P.ksplit_ok = (lid == HA2 || lid == HA3 || lid == HS1) && P.halo && !P.wres && (P.tps == 2 || P.tps == 3) &&
                      P.cg == 2 && P.n_ntiles == 1 && (Ly.ep == EP_RELU || Ly.ep == EP_ZQUANT) && P.Cout % 8 == 0;
    }
    P.L = c->L;
    P.no_guard = (Ly.y_bounded && c->no_guard_enabled) ? 1 : 0;
    // tensor maps
    const int ntaps_w = (gemm_l1 || P.gather) ? 1 : (P.pack4 ? 9 : Ly.k * Ly.k);
    const int cout_pad = P.BN * P.n_ntiles;
    if (!P.fuse_l1 && !encode_act_map(&Ly.mapA, Ly.in_buf, P.Cin, Ly.deconv ? Ly.Win : (gemm_l1 ? Ly.Wout : Ly.Win),
                        Ly.deconv ? Ly.Hin : (gemm_l1 ? Ly.Hout : Ly.Hin), c->max_batch, P.split, Ly.in_plane,
                        P.halo ? P.halo_w : P.Wt, P.halo ? P.Ht + 2 : P.Ht, P.stride))
        return fail(c, LIC_ECUDA, "cuTensorMapEncodeTiled (activations) failed");
    if (!encode_w_map(&Ly.mapB, Ly.w, P.Cin, cout_pad, ntaps_w, P.BN / P.cg))
        return fail(c, LIC_ECUDA, "cuTensorMapEncodeTiled (weights) failed");
    if (gdn) {
        if (!encode_w_map(&Ly.mapG, Ly.gamma, Ly.Cout, Ly.Cout, 1, Ly.Cout / P.cg))
            return fail(c, LIC_ECUDA, "cuTensorMapEncodeTiled (gamma) failed");
    } else {
        Ly.mapG = Ly.mapB;
    }
    Ly.mapOH = Ly.mapB;
    Ly.mapOL = Ly.mapB;
    Ly.mapO2 = Ly.mapB;
    Ly.mapO3 = Ly.mapB;
    if (P.tma_out) {
        const int bw = P.Wt < 32 ? P.Wt : 32, bh = 32 / bw;
        const int bc = P.wst_ch ? P.wst_ch : 64;
        bool ok;
        if (P.wst_ch && P.nphase == 1)
            ok = encode_out_conv_map_pl(&Ly.mapOH, Ly.out_buf, Ly.Cout, Ly.Wout, Ly.Hout, c->max_batch, Ly.out_plane,
                                        P.split, bw, bh, bc);
        else if (P.wst_ch) {
            CUtensorMap* pm[4] = {&Ly.mapOH, &Ly.mapOL, &Ly.mapO2, &Ly.mapO3};
            ok = true;
            for (int ph = 0; ph < 4 && ok; ++ph)
                ok = encode_out_phase_map_pl(pm[ph], Ly.out_buf, Ly.Cout, Ly.Wout, Ly.Hout, c->max_batch, Ly.out_plane,
                                             P.split, ph, bw, bh, bc);
        } else if (P.nphase == 1)
            ok = encode_out_conv_map(&Ly.mapOH, Ly.out_buf, Ly.Cout, Ly.Wout, Ly.Hout, c->max_batch, bw, bh, bc) &&
                 encode_out_conv_map(&Ly.mapOL, Ly.out_buf + Ly.out_plane, Ly.Cout, Ly.Wout, Ly.Hout, c->max_batch, bw, bh,
                                     bc);
        else
            ok = encode_out_phase_map(&Ly.mapOH, Ly.out_buf, Ly.Cout, Ly.Wout, Ly.Hout, c->max_batch, bw, bh, bc) &&
                 encode_out_phase_map(&Ly.mapOL, Ly.out_buf + Ly.out_plane, Ly.Cout, Ly.Wout, Ly.Hout, c->max_batch, bw,
                                      bh, bc);
        if (!ok) return fail(c, LIC_ECUDA, "cuTensorMapEncodeTiled (output) failed");
    }
    // epilogue constants
    P.ep = Ly.ep;
    P.Hout = Ly.Hout;
    P.Wout = Ly.Wout;
    P.bias = Ly.bias;
    P.beta = Ly.beta;
    P.table = c->table;
    P.out_act = Ly.out_buf;
    P.act_plane = Ly.out_plane;
    P.crop_top = 0; P.crop_left = 0; P.crop_H = Ly.Hout; P.crop_W = Ly.Wout;
    if (std::getenv("LIC_PLAN_DEBUG"))
        std::fprintf(stderr, "plan layer %d: BN %d cg %d ntiles %d halo %d sub4 %d tps %d stages %d slots %d wres %d "
                     "tma_out %d ostage %d smem %u kchunks %d wst %d/%d\n", lid_of(c, Ly), P.BN, P.cg,
                     P.n_ntiles, P.halo, P.sub4, P.tps, P.stages, P.halo_slots, P.wres, P.tma_out, P.ostage_slots,
                     P.smem_bytes, P.kchunks, P.wst_ch, P.wst_slots);
    return LIC_OK;
}

static lic_status run_layer(lic_codec* c, Layer& Ly, const ConvParams& P0, int batch, cudaStream_t st,
                            const CUtensorMap* mapA = nullptr) {
    ConvParams P = P0;
    P.batch = batch;
    const int txs = (P.tiles_x + P.cg - 1) / P.cg;          // tiles (or CTA-pair tiles) along x
    P.total_tiles = batch * P.nphase * P.tiles_y * txs * P.n_ntiles;
    // split-K: a layer with fewer (pair) tiles than a quarter of the SMs runs each
    // tile as S K slices on S times as many CTAs; the slices' fp32 partial sums are added in
    // slice order by split_reduce_kernel, which applies the layer's epilogue
    int S = 1;
    if (P.ksplit_ok && c->ksplit_enabled && c->d_part) {
        S = std::min(kKsplitMax, (c->num_sms / P.cg) / std::max(1, P.total_tiles));
        if (c->ksplit_force) S = std::min(S, c->ksplit_force);
        if (S < 2) S = 1;
    }
    const ConvParams Pe = P;                                   // the layer's own epilogue fields
    P.ksplit = S;
    if (S > 1) {
        P.total_tiles *= S;
        P.ep = EP_PARTIAL;
        P.part = c->d_part;
        P.out_act = nullptr; P.out_sym = nullptr; P.out_f32 = nullptr;
        P.sat_count = nullptr; P.range_count = nullptr;
        P.tma_out = 0;
    }
    const int grid = P.cg * std::min(P.total_tiles, c->num_sms / P.cg);
    const int lid = lid_of(c, Ly);
    P.pdl = c->pdl_enabled;
    if (c->trace_layer == lid && c->d_trace) {
        P.trace = c->d_trace;
        if (const char* e = std::getenv("LIC_DBG_NOSTORE")) P.dbg_nostore = atoi(e);
        CK(cudaMemsetAsync(c->d_trace, 0, 256 * kTraceEvents * 8, st));
    }
    const bool prof = c->profiling && ((c->prof_mask >> lid) & 1u);
    if (prof) {
        if (c->ev_used == kProfSlots) prof_flush(c);
        CK(cudaEventRecord(c->ev[2 * c->ev_used], st));
    }
    {
        const cudaError_t e = launch_conv_umma(mapA ? *mapA : Ly.mapA, Ly.mapB, Ly.mapG, Ly.mapOH, Ly.mapOL, Ly.mapO2, Ly.mapO3, P,
                                               grid, st);
        if (e != cudaSuccess)
            return fail(c, LIC_ECUDA, "launch of layer %d (grid %d, cg %d, smem %u, tiles %d, stages %d, halo %d): %s",
                        lid, grid, P.cg, P.smem_bytes, P.total_tiles, P.stages, P.halo, cudaGetErrorString(e));
    }
    ++c->launches;
    if (S > 1) {
        const cudaError_t e = launch_split_reduce(c->d_part, S, batch, Pe.Hout, Pe.Wout, Pe.Cout, Pe.bias, Pe.mu, Pe.ep,
                                                  Pe.L, reinterpret_cast<__half*>(Pe.out_act), Pe.act_plane, Pe.split,
                                                  reinterpret_cast<int8_t*>(Pe.out_sym), Pe.out_f32, Pe.sat_count,
                                                  Pe.range_count, st);
        if (e != cudaSuccess) return fail(c, LIC_ECUDA, "split-K reduce of layer %d: %s", lid, cudaGetErrorString(e));
        ++c->launches;
    }
    if (prof) {
        CK(cudaEventRecord(c->ev[2 * c->ev_used + 1], st));
        c->ev_layer[c->ev_used++] = lid;
    }
    return LIC_OK;
}

// ------------------------------------------------------------------ pointer handling
struct OutBuf { void* dev; void* user; size_t bytes; };
static void* device_only(const void* p);
// Returns a device-accessible alias of p (device memory or pinned/mapped host memory),
// or nullptr if p is pageable host memory that must be staged.
static void* device_alias(const void* p) {
    if (!p) return nullptr;
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) { cudaGetLastError(); return nullptr; }
    if (a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged) return const_cast<void*>(p);
    if (a.type == cudaMemoryTypeHost && a.devicePointer) return a.devicePointer;
    return nullptr;
}

// Device memory only (frames: host frames are moved by DMA into the staging buffer, since the
// ingest gather and the per-channel frame stores would be uncoalesced over PCIe).
static void* device_only(const void* p) {
    if (!p) return nullptr;
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) { cudaGetLastError(); return nullptr; }
    if (a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged) return const_cast<void*>(p);
    return nullptr;
}

static OutBuf route_frames_out(void* user, void* staging, size_t bytes) {
    void* d = device_only(user);
    return d ? OutBuf{d, nullptr, bytes} : OutBuf{staging, user, bytes};
}

// ------------------------------------------------------------------ ABI
extern "C" const char* lic_version(void) { return "lic-b200 0.1 (sm_100a tcgen05)"; }

// lic_open's failures have no codec to hold the message: a thread-local one instead
static thread_local std::string g_open_err;

extern "C" const char* lic_last_error(const lic_codec* c) { return c ? c->err.c_str() : g_open_err.c_str(); }

extern "C" void lic_close(lic_codec* c) {
    if (!c) return;
    cudaSetDevice(c->device);
    if (c->stream) cudaStreamSynchronize(c->stream);
    for (cudaEvent_t e : c->ev) cudaEventDestroy(e);
    for (void* p : c->allocs) cudaFree(p);
    if (c->ws_own) cudaFree(c->ws_own);
    {
        std::lock_guard<std::mutex> g(c->pool_mu);
        for (auto& kv : c->owned) cudaFreeHost(kv.first);
    }
    if (c->stream) cudaStreamDestroy(c->stream);
    delete c;
}

// ------------------------------------------------------------------ workspace
// Everything whose size follows the batch: the activation ping-pong buffers A / B (fp16 hi +
// lo NHWC planes of the largest activation, Hp/2 x Wp/2 x N), the y-plane (|y| or y-hat), the
// z-plane (z-hat), the host-frame staging buffer and the symbol / index staging planes.  One
// block, carved in this order at 256-byte boundaries; owned by the library (lic_open) or by
// the caller (lic_bind_workspace).
// (hyperprior codecs add the split-K partial sums of the h layers: fp32 [kKsplitMax][B][Hp/32][Wp/32][N])
struct WsLayout { size_t planeA, planeY, planeZ, off[9], total; };
static WsLayout ws_layout(const lic_codec* c, int B) {
    WsLayout L{};
    const int S = c->split, N = c->N, M = c->M;
    const size_t Hy = c->Hp / 16, Wy = c->Wp / 16, Hz = std::max(1, c->Hp / 64), Wz = std::max(1, c->Wp / 64);
    L.planeA = (size_t)B * (c->Hp / 2) * (c->Wp / 2) * N;
    L.planeY = (size_t)B * Hy * Wy * M;
    L.planeZ = (size_t)B * Hz * Wz * N;
    const size_t npart = c->kind == 1 ? (size_t)kKsplitMax * B * (c->Hp / 32) * (c->Wp / 32) * N * 4 : 0;
    const size_t sz[9] = {L.planeA * S * 2, L.planeA * S * 2, L.planeY * S * 2, L.planeZ * S * 2,
                          (size_t)B * 3 * c->H * c->W * 4, (size_t)B * M * Hy * Wy, (size_t)B * M * Hy * Wy,
                          (size_t)B * N * Hz * Wz, npart};
    size_t o = 0;
    for (int i = 0; i < 9; ++i) { L.off[i] = o; o += (sz[i] + 255) / 256 * 256; }
    L.total = o;
    return L;
}
static void ws_carve(lic_codec* c, uint8_t* base, int B) {
    const WsLayout L = ws_layout(c, B);
    c->planeA = L.planeA; c->planeY = L.planeY; c->planeZ = L.planeZ;
    c->bufA = (__half*)(base + L.off[0]);
    c->bufB = (__half*)(base + L.off[1]);
    c->bufY = (__half*)(base + L.off[2]);
    c->bufZ = (__half*)(base + L.off[3]);
    c->d_frames = base + L.off[4];
    c->d_ysym = (int8_t*)(base + L.off[5]);
    c->d_yidx = (uint8_t*)(base + L.off[6]);
    c->d_zsym = (int8_t*)(base + L.off[7]);
    c->d_part = c->kind == 1 ? (float*)(base + L.off[8]) : nullptr;
}
static __half* ws_buf(const lic_codec* c, char id, size_t* plane) {
    switch (id) {
    case 'A': *plane = c->planeA; return c->bufA;
    case 'B': *plane = c->planeA; return c->bufB;
    case 'Y': *plane = c->planeY; return c->bufY;
    case 'Z': *plane = c->planeZ; return c->bufZ;
    default: *plane = 0; return nullptr;
    }
}

static lic_status upload(lic_codec* c, void* dst, const void* src, size_t bytes) {
    CK(cudaMemcpy(dst, src, bytes, cudaMemcpyHostToDevice));
    return LIC_OK;
}

// per-codec epilogue settings of the layer plans (after plan_layer)
// alternative plans of two layers, copies of the layer (weights, buffers) planned differently and
// picked per call: g_s L1 with a hi-only halo ring (the hyperprior's integer y-hat, decode_impl)
// and g_a L1 in row-halo mode (l1_rows; encode_impl, when the frames are u8 with 16-byte rows)
static lic_status plan_variants(lic_codec* c) {
    c->gs1h_ok = false;
    if (c->layers[GS1].present && c->kind == 1 && c->a_hi_only_enabled && c->gs1_hi_plan && c->layers[GS1].prm.halo) {
        c->gs1h = c->layers[GS1];
        if (lic_status r = plan_layer(c, c->gs1h)) return r;
        c->gs1h_ok = c->gs1h.prm.halo == 1;
    }
    c->l1r_ok = false;
    if (!c->layers[GA1].present || !c->l1_rows_enabled) return LIC_OK;
    c->l1r = c->layers[GA1];
    if (lic_status r = plan_layer(c, c->l1r)) return r;
    c->l1r_ok = true;
    return LIC_OK;
}

static void finish_plans(lic_codec* c) {
    for (int l = 0; l < NLAYER; ++l)
        if (c->layers[l].present) c->layers[l].prm.range_count = c->d_range;
    c->layers[GA4].prm.mu = c->kind == 0 ? c->mu_y : nullptr;
    c->layers[GA4].prm.abs_out = c->kind == 1;
    for (int l : {GA1, GA2, GA3, GS1, GS2, GS3}) c->layers[l].prm.onedn = c->act == 1;
    if (c->kind == 1) c->layers[HA3].prm.mu = c->mu_z;
    c->layers[GS4].prm.crop_top = c->top;
    c->layers[GS4].prm.crop_left = c->left;
    c->layers[GS4].prm.crop_H = c->H;
    c->layers[GS4].prm.crop_W = c->W;
    if (c->l1r_ok) {
        c->l1r.prm.range_count = c->d_range;
        c->l1r.prm.onedn = c->act == 1;
    }
    if (c->gs1h_ok) {
        c->gs1h.prm.range_count = c->d_range;
        c->gs1h.prm.onedn = c->act == 1;
    }
}

extern "C" lic_status lic_open(const uint8_t* licw, size_t len, int device, uint32_t height, uint32_t width,
                               uint32_t max_batch, int precision, lic_codec** out) {
    g_open_err.clear();
    if (!licw || !out || max_batch == 0) return LIC_EINVAL;
    *out = nullptr;
    if (height == 0 || width == 0 || height > 8192 || width > 8192) return LIC_ESHAPE;
    if (precision != LIC_PREC_SPLIT && precision != LIC_PREC_F16) return LIC_EINVAL;
    if (len < 13 || std::memcmp(licw, "LICW", 4) != 0 || licw[4] != 1) return LIC_EDIGEST;
    lic_codec* c = new lic_codec();
    auto bail = [&](lic_status st) {
        if (g_open_err.empty() && !c->err.empty()) g_open_err = c->err;
        lic_close(c);
        return st;
    };
    c->licw.assign(licw, licw + len);
    c->precision = precision;
    c->kind = licw[5];
    c->act = licw[6];
    c->N = rd<uint16_t>(licw + 7);
    c->M = rd<uint16_t>(licw + 9);
    c->L = rd<uint16_t>(licw + 11);
    if (c->kind > 1 || c->act > 1) return bail(LIC_EINVAL);       // act 0 GDN, 1 1DN
    if (c->N % 64 || c->M % 64 || c->N < 64 || c->N > 256 || c->M < 64 || c->M > 512 || c->L < 1 || c->L > 127)
        return bail(LIC_EINVAL);
    // ---- parse blocks
    std::map<std::string, std::vector<float>> blk;
    size_t off = 13;
    for (const BlockSpec& b : licw_blocks(c->N, c->M)) {
        if (b.hyper_only && c->kind != 1) continue;
        size_t cnt = 1;
        for (int d : b.shape) cnt *= (size_t)d;
        if (off + 5 > len || licw[off] != b.tag || rd<uint32_t>(licw + off + 1) != cnt) return bail(LIC_EDIGEST);
        off += 5;
        if (off + 4 * cnt > len) return bail(LIC_EDIGEST);
        std::vector<float> v(cnt);
        std::memcpy(v.data(), licw + off, 4 * cnt);
        off += 4 * cnt;
        for (float f : v)
            if (!std::isfinite(f)) return bail(LIC_EINVAL);
        if (b.role == R_BETA)
            for (float f : v) if (!(f > 0.0f)) return bail(LIC_EINVAL);
        if (b.role == R_GAMMA)
            for (float f : v) if (!(f >= 0.0f)) return bail(LIC_EINVAL);
        // The tensor cores multiply fp16 operands: conv / deconv weights and gamma must be
        // exactly representable in fp16 (the split-FP16 precision, R16; the paper's
        // FP16 engines hold fp16 weights too).  Rounding them here would miss
        // the oracle's parity bar silently, so a container with other values is rejected.
        if (b.role == R_CONV || b.role == R_DECONV || b.role == R_GAMMA)
            for (size_t i = 0; i < v.size(); ++i)
                if (__half2float(__float2half_rn(v[i])) != v[i]) {
                    char m[160];
                    std::snprintf(m, sizeof m, "%s[%zu] = %.9g is not exactly representable in fp16", b.name.c_str(), i,
                                  (double)v[i]);
                    g_open_err = m;
                    return bail(LIC_EINVAL);
                }
        blk[b.name] = std::move(v);
    }
    if (off != len) return bail(LIC_EDIGEST);
    const std::vector<float>& tab = blk["scale_table"];
    for (int i = 1; i < 64; ++i) if (!(tab[i] > tab[i - 1]) || !(tab[0] > 0)) return bail(LIC_EINVAL);

    // ---- device
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || device < 0 || device >= ndev) {
        cudaGetLastError();
        return bail(LIC_ECUDA);
    }
    cudaDeviceProp prop;
    if (cudaSetDevice(device) != cudaSuccess || cudaGetDeviceProperties(&prop, device) != cudaSuccess ||
        prop.major != 10) {
        cudaGetLastError();
        return bail(LIC_ECUDA);
    }
    if (!get_encode_fn()) return bail(LIC_ECUDA);
    c->device = device;
    c->num_sms = prop.multiProcessorCount;
    if (cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking) != cudaSuccess) return bail(LIC_ECUDA);
    c->split = precision == LIC_PREC_SPLIT ? 2 : 1;
    if (const char* e = std::getenv("LIC_NO_HALO")) c->halo_enabled = (e[0] == '0');
    if (const char* e = std::getenv("LIC_TMA_OUT")) c->tma_out_enabled = (e[0] != '0');
    if (const char* e = std::getenv("LIC_CG")) c->cg_enabled = (e[0] != '1');
    if (const char* e = std::getenv("LIC_GS4_BN")) c->gs4_bn = (atoi(e) == 16) ? 16 : 32;
    if (const char* e = std::getenv("LIC_PDL")) c->pdl_enabled = (e[0] != '0');
    if (const char* e = std::getenv("LIC_GS4_GATHER")) c->gs4_gather = (e[0] != '0');
    if (const char* e = std::getenv("LIC_L1_INT")) c->l1_int_enabled = (e[0] != '0');
    if (const char* e = std::getenv("LIC_G2")) c->g2_enabled = atoi(e);      // 0 off, 1 g_a L1, 2 every BN = 128 GDN layer
    if (const char* e = std::getenv("LIC_L1_STAGES")) c->l1_stage_split = (e[0] != '0');
    if (const char* e = std::getenv("LIC_RAW_TMA")) c->raw_tma_enabled = (e[0] != '0');
    if (const char* e = std::getenv("LIC_MMA_SPIN")) c->mma_spin = (e[0] == '1');
    if (const char* e = std::getenv("LIC_G2_192")) c->g2_192 = (e[0] != '0');
    if (const char* e = std::getenv("LIC_G2_SLOT16")) c->g2_slot16 = (e[0] != '0');
    if (const char* e = std::getenv("LIC_KSPLIT")) { c->ksplit_enabled = atoi(e) != 0; c->ksplit_force = atoi(e) > 1 ? atoi(e) : 0; }
    if (const char* e = std::getenv("LIC_L1_CONV")) c->l1_conv_enabled = (e[0] != '0');
    if (const char* e = std::getenv("LIC_L1_ROWS")) c->l1_rows_enabled = (e[0] != '0');
    if (const char* e = std::getenv("LIC_G2_DB16")) c->g2_db16 = atoi(e);
    if (const char* e = std::getenv("LIC_GS1_HI")) c->gs1_hi_plan = (e[0] != '0');
    if (const char* e = std::getenv("LIC_NO_GUARD")) c->no_guard_enabled = (e[0] != '0');
    if (const char* e = std::getenv("LIC_YHAT_HI")) c->a_hi_only_enabled = (e[0] != '0');
    if (const char* e = std::getenv("LIC_S2HALO")) c->s2halo_enabled = (e[0] != '0');
    if (const char* e = std::getenv("LIC_HS3_SPLITN")) c->hs3_split_n = (e[0] != '0');
    if (const char* e = std::getenv("LIC_SMALL_BN")) c->small_bn = atoi(e) == 64 || atoi(e) == 96 || atoi(e) == 128 ? atoi(e) : 0;
    if (const char* e = std::getenv("LIC_NO_WRES")) c->wres_enabled = (e[0] != '1');
    if (const char* e = std::getenv("LIC_WSTAGE")) c->wstage_enabled = (e[0] != '0');
    c->max_batch = (int)max_batch;
    c->H = (int)height; c->W = (int)width;
    const int P = c->kind == 1 ? 64 : 16;
    c->Hp = (c->H + P - 1) / P * P; c->Wp = (c->W + P - 1) / P * P;
    c->top = (c->Hp - c->H) / 2; c->left = (c->Wp - c->W) / 2;
    const int N = c->N, M = c->M, B = c->max_batch, S = c->split;
    const int H2 = c->Hp / 2, W2 = c->Wp / 2, Hy = c->Hp / 16, Wy = c->Wp / 16, Hz = c->Hp / 64, Wz = c->Wp / 64;

    // ---- host tables (CDF build)
    c->h_table = tab;
    c->h_mu_y = blk["mu_y"];
    c->h_sigma_y = blk["sigma_y"];
    const uint32_t rl = 2 * c->L + 2;
    if (c->kind == 0) {
        c->cdf_fact.resize((size_t)M * rl);
        if (lic_cdf_build(c->h_sigma_y.data(), M, c->L, c->cdf_fact.data()) != LIC_OK) return bail(LIC_EINVAL);
    } else {
        c->h_mu_z = blk["mu_z"];
        c->h_sigma_z = blk["sigma_z"];
        c->cdf_z.resize((size_t)N * rl);
        c->cdf_gauss.resize((size_t)64 * rl);
        if (lic_cdf_build(c->h_sigma_z.data(), N, c->L, c->cdf_z.data()) != LIC_OK ||
            lic_cdf_build(tab.data(), 64, c->L, c->cdf_gauss.data()) != LIC_OK)
            return bail(LIC_EINVAL);
    }

    // ---- workspace (activation planes of fp16 NHWC, staging) -- one block, re-bindable
    c->open_batch = B;
    c->ws_bytes = ws_layout(c, B).total;
    if (cudaMalloc(&c->ws_own, c->ws_bytes) != cudaSuccess) {
        cudaGetLastError();
        c->ws_own = nullptr;
        return bail(fail(c, LIC_ENOMEM, "cudaMalloc(%zu) failed (workspace)", c->ws_bytes));
    }
    ws_carve(c, (uint8_t*)c->ws_own, B);
    lic_status st;
    if ((st = dalloc(c, &c->table, 64 * 4)) || (st = dalloc(c, &c->mu_y, (size_t)M * 4)) ||
        (st = dalloc(c, &c->mu_z, (size_t)N * 4)) || (st = dalloc(c, &c->d_sat, 8)) || (st = dalloc(c, &c->d_range, 8)))
        return bail(st);
    if ((st = upload(c, c->table, tab.data(), 256)) || (st = upload(c, c->mu_y, c->h_mu_y.data(), (size_t)M * 4)))
        return bail(st);
    if (c->kind == 1 && (st = upload(c, c->mu_z, c->h_mu_z.data(), (size_t)N * 4))) return bail(st);

    // ---- layers
    struct Def { int id; bool deconv; int k, s, p, cin, cout, hin, win, hout, wout; EpKind ep; char in, out; };
    std::vector<Def> defs = {
        {GA1, false, 5, 2, 2, 3, N, c->Hp, c->Wp, H2, W2, EP_GDN, 0, 'A'},
        {GA2, false, 5, 2, 2, N, N, H2, W2, H2 / 2, W2 / 2, EP_GDN, 'A', 'B'},
        {GA3, false, 5, 2, 2, N, N, H2 / 2, W2 / 2, H2 / 4, W2 / 4, EP_GDN, 'B', 'A'},
        {GA4, false, 5, 2, 2, N, M, H2 / 4, W2 / 4, Hy, Wy, EP_YQUANT, 'A', 'Y'},
        {GS1, true, 5, 2, 2, M, N, Hy, Wy, Hy * 2, Wy * 2, EP_IGDN, 'Y', 'A'},
        {GS2, true, 5, 2, 2, N, N, Hy * 2, Wy * 2, Hy * 4, Wy * 4, EP_IGDN, 'A', 'B'},
        {GS3, true, 5, 2, 2, N, N, Hy * 4, Wy * 4, H2, W2, EP_IGDN, 'B', 'A'},
        {GS4, true, 5, 2, 2, N, 3, H2, W2, c->Hp, c->Wp, EP_FINAL, 'A', 0},
    };
    if (c->kind == 1) {
        defs.push_back({HA1, false, 3, 1, 1, M, N, Hy, Wy, Hy, Wy, EP_RELU, 'Y', 'A'});
        defs.push_back({HA2, false, 5, 2, 2, N, N, Hy, Wy, Hy / 2, Wy / 2, EP_RELU, 'A', 'B'});
        defs.push_back({HA3, false, 5, 2, 2, N, N, Hy / 2, Wy / 2, Hz, Wz, EP_ZQUANT, 'B', 'Z'});
        defs.push_back({HS1, true, 5, 2, 2, N, N, Hz, Wz, Hz * 2, Wz * 2, EP_RELU, 'Z', 'A'});
        defs.push_back({HS2, true, 5, 2, 2, N, N, Hz * 2, Wz * 2, Hy, Wy, EP_RELU, 'A', 'B'});
        defs.push_back({HS3, false, 3, 1, 1, N, M, Hy, Wy, Hy, Wy, EP_SIGMA, 'B', 0});
    }
    size_t dbg = 0;
    for (const Def& d : defs) {
        Layer& Ly = c->layers[d.id];
        Ly.present = true;
        Ly.deconv = d.deconv; Ly.k = d.k; Ly.s = d.s; Ly.p = d.p;
        Ly.Cin = d.cin; Ly.Cout = d.cout;
        Ly.Cin_eff = d.id == GA1 ? 128 : d.cin;
        Ly.Hin = d.hin; Ly.Win = d.win; Ly.Hout = d.hout; Ly.Wout = d.wout;
        Ly.ep = d.ep;
        Ly.in_id = d.in; Ly.out_id = d.out;
        Ly.in_buf = ws_buf(c, d.in, &Ly.in_plane);
        Ly.out_buf = ws_buf(c, d.out, &Ly.out_plane);
        dbg = std::max(dbg, (size_t)B * d.cout * d.hout * d.wout);
        dbg = std::max(dbg, (size_t)B * d.cin * d.hin * d.win);
        // weights: LICW out x in x k x k (fp32, fp16-exact) -> fp16 [tap][co_pad][ci_eff]
        const std::string wn = std::string(kLayerW[d.id]);
        const std::vector<float>& w = blk[wn + ".w"];
        int bn = d.cout <= 256 ? (d.cout + 15) / 16 * 16 : 0;
        if (!bn) { int nt = (d.cout + 255) / 256; bn = ((d.cout + nt - 1) / nt + 15) / 16 * 16 * nt; }
        const bool gather = d.id == GS4 && c->gs4_gather;
        const bool pack4 = d.id == GS4 && !gather;
        const int cout_pad = gather ? kGatherN : pack4 ? c->gs4_bn : bn;
        const int taps = (d.id == GA1 || gather) ? 1 : (pack4 ? 9 : d.k * d.k);
        std::vector<__half> wp((size_t)taps * cout_pad * Ly.Cin_eff, __float2half(0.0f));
        if (gather) {
            // row t*16 + phase*4 + co, t = (dy+1)*3 + (dx+1): the tap of sub-pixel phase (py, px)
            // that reads input offset (dy, dx) (ky = py + 2 - 2dy, kx = px + 2 - 2dx)
            for (int t = 0; t < 9; ++t) {
                const int dy = t / 3 - 1, dx = t % 3 - 1;
                for (int ph = 0; ph < 4; ++ph) {
                    const int ky = (ph >> 1) + 2 - 2 * dy, kx = (ph & 1) + 2 - 2 * dx;
                    if (ky < 0 || ky > 4 || kx < 0 || kx > 4) continue;
                    for (int co = 0; co < 3; ++co)
                        for (int ci = 0; ci < d.cin; ++ci)
                            wp[((size_t)t * 16 + ph * 4 + co) * Ly.Cin_eff + ci] =
                                __float2half_rn(w[(((size_t)co * d.cin + ci) * 5 + ky) * 5 + kx]);
                }
            }
        }
        if (pack4) {
            for (int t = 0; t < 9; ++t) {
                const int dy = t / 3 - 1, dx = t % 3 - 1;
                for (int ph = 0; ph < 4; ++ph) {
                    const int ky = (ph >> 1) + 2 - 2 * dy, kx = (ph & 1) + 2 - 2 * dx;
                    if (ky < 0 || ky > 4 || kx < 0 || kx > 4) continue;
                    for (int co = 0; co < 3; ++co)
                        for (int ci = 0; ci < d.cin; ++ci)
                            wp[((size_t)t * cout_pad + ph * 4 + co) * Ly.Cin_eff + ci] =
                                __float2half_rn(w[(((size_t)co * d.cin + ci) * 5 + ky) * 5 + kx]);
                }
            }
        }
        for (int co = 0; co < d.cout && !pack4 && !gather; ++co)
            for (int ci = 0; ci < d.cin; ++ci)
                for (int ky = 0; ky < d.k; ++ky)
                    for (int kx = 0; kx < d.k; ++kx) {
                        const float v = w[(((size_t)co * d.cin + ci) * d.k + ky) * d.k + kx];
                        size_t o;
                        if (d.id == GA1) o = (size_t)co * 128 + ky * 16 + kx * 3 + ci;      // fused im2col K order
                        else o = ((size_t)(ky * d.k + kx) * cout_pad + co) * Ly.Cin_eff + ci;
                        wp[o] = __float2half_rn(v);
                    }
        if ((st = dalloc(c, &Ly.w, wp.size() * 2)) || (st = upload(c, Ly.w, wp.data(), wp.size() * 2))) return bail(st);
        const std::vector<float>& bb = blk[wn + ".b"];
        if ((st = dalloc(c, &Ly.bias, bb.size() * 4)) || (st = upload(c, Ly.bias, bb.data(), bb.size() * 4)))
            return bail(st);
        if (d.ep == EP_GDN || d.ep == EP_IGDN) {
            const std::vector<float>& be = blk[wn + ".beta"];
            const std::vector<float>& ga = blk[wn + ".gamma"];
            std::vector<__half> gh(ga.size());
            for (size_t i = 0; i < ga.size(); ++i) gh[i] = __float2half_rn(ga[i]);
            // forward GDN / 1DN output bound (R16f): with gamma >= 0 and beta >= 0,
            // n_i >= gamma_ii x_i^2 (GDN) / gamma_ii |x_i| (1DN), so |y_i| <= 1 / sqrt(gamma_ii) resp.
            // 1 / gamma_ii -- below 60000 (fp16 range, rounding margin) the range guard cannot fire
            if (d.ep == EP_GDN) {
                const int n = Ly.Cout;
                bool ok = true;
                for (size_t i = 0; i < gh.size() && ok; ++i) ok = __half2float(gh[i]) >= 0.0f;
                for (size_t i = 0; i < be.size() && ok; ++i) ok = be[i] >= 0.0f;
                for (int i = 0; i < n && ok; ++i) {
                    const double g = __half2float(gh[(size_t)i * n + i]);
                    ok = c->act == 1 ? g >= 1.0 / 60000.0 : g >= 1.0 / (60000.0 * 60000.0);
                }
                Ly.y_bounded = ok;
            }
            if ((st = dalloc(c, &Ly.beta, be.size() * 4)) || (st = upload(c, Ly.beta, be.data(), be.size() * 4)) ||
                (st = dalloc(c, &Ly.gamma, gh.size() * 2)) || (st = upload(c, Ly.gamma, gh.data(), gh.size() * 2)))
                return bail(st);
        }
        if ((st = plan_layer(c, Ly))) return bail(st);
    }
    if ((st = plan_variants(c))) return bail(st);
    if (cudaMemset(c->d_range, 0, 8) != cudaSuccess) return bail(LIC_ECUDA);
    finish_plans(c);
    c->dbg_elems = dbg;
    *out = c;
    return LIC_OK;
}

extern "C" size_t lic_workspace_bytes(const lic_codec* c, uint32_t batch) {
    if (!c) return 0;
    if (batch == 0) batch = (uint32_t)c->open_batch;
    if ((int)batch > c->open_batch) return 0;
    return ws_layout(c, (int)batch).total;
}

extern "C" lic_status lic_bind_workspace(lic_codec* c, void* dev_ptr, size_t bytes) {
    if (!c || !dev_ptr) return LIC_EINVAL;
    if (c->sticky) return LIC_ECUDA;
    if ((uintptr_t)dev_ptr % 256) return fail(c, LIC_EINVAL, "workspace must be 256-byte aligned");
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, dev_ptr) != cudaSuccess || a.type != cudaMemoryTypeDevice || a.device != c->device) {
        cudaGetLastError();
        return fail(c, LIC_EINVAL, "workspace is not device memory of device %d", c->device);
    }
    // the largest batch the block holds (planes scale with the batch)
    int b = c->open_batch;
    while (b > 0 && ws_layout(c, b).total > bytes) --b;
    if (b == 0) return fail(c, LIC_ENOSPACE, "workspace of %zu bytes < %zu for one frame", bytes, ws_layout(c, 1).total);
    CK(cudaSetDevice(c->device));
    CK(cudaDeviceSynchronize());                 // nothing may still use the old block
    const int old_batch = c->max_batch;
    c->max_batch = b;
    ws_carve(c, (uint8_t*)dev_ptr, b);
    for (int l = 0; l < NLAYER; ++l) {
        Layer& Ly = c->layers[l];
        if (!Ly.present) continue;
        Ly.in_buf = ws_buf(c, Ly.in_id, &Ly.in_plane);
        Ly.out_buf = ws_buf(c, Ly.out_id, &Ly.out_plane);
        lic_status r = plan_layer(c, Ly);        // tensor maps over the new planes
        if (r) { c->max_batch = old_batch; c->sticky = true; return r; }
    }
    if (lic_status r = plan_variants(c)) { c->max_batch = old_batch; c->sticky = true; return r; }
    finish_plans(c);
    if (c->ws_own) { cudaFree(c->ws_own); c->ws_own = nullptr; }
    c->ws_user = dev_ptr;
    c->ws_bytes = ws_layout(c, b).total;
    return LIC_OK;
}

extern "C" lic_status lic_max_batch(const lic_codec* c, uint32_t* max_batch) {
    if (!c || !max_batch) return LIC_EINVAL;
    *max_batch = (uint32_t)c->max_batch;
    return LIC_OK;
}

extern "C" lic_status lic_shapes(const lic_codec* c, lic_shape* y, lic_shape* z, int* kind) {
    if (!c) return LIC_EINVAL;
    if (y) *y = {(uint32_t)c->M, (uint32_t)(c->Hp / 16), (uint32_t)(c->Wp / 16)};
    if (z) *z = c->kind == 1 ? lic_shape{(uint32_t)c->N, (uint32_t)(c->Hp / 64), (uint32_t)(c->Wp / 64)}
                             : lic_shape{0, 0, 0};
    if (kind) *kind = c->kind;
    return LIC_OK;
}

extern "C" lic_status lic_layer_shapes(const lic_codec* c, int id, lic_shape* in, lic_shape* out) {
    if (!c || id < 0 || id >= NLAYER || !c->layers[id].present) return LIC_EINVAL;
    const Layer& L = c->layers[id];
    if (in) *in = {(uint32_t)L.Cin, (uint32_t)L.Hin, (uint32_t)L.Win};
    if (out) *out = {(uint32_t)L.Cout, (uint32_t)L.Hout, (uint32_t)L.Wout};
    return LIC_OK;
}

extern "C" lic_status lic_cdf(const lic_codec* c, int which, const uint32_t** rows, uint32_t* n_rows,
                              uint32_t* row_len) {
    if (!c || !rows || !n_rows || !row_len) return LIC_EINVAL;
    const std::vector<uint32_t>* t = which == 0 ? &c->cdf_fact : which == 1 ? &c->cdf_z : which == 2 ? &c->cdf_gauss : nullptr;
    if (!t || t->empty()) return LIC_EINVAL;
    *row_len = 2 * c->L + 2;
    *n_rows = (uint32_t)(t->size() / *row_len);
    *rows = t->data();
    return LIC_OK;
}

extern "C" lic_status lic_sigmas(const lic_codec* c, int which, const float** sig, uint32_t* n) {
    if (!c || !sig || !n) return LIC_EINVAL;
    const std::vector<float>* t = which == 0 ? &c->h_sigma_y : which == 1 ? &c->h_sigma_z : which == 2 ? &c->h_table : nullptr;
    if (!t || t->empty() || (which == 0 && c->kind != 0) || (which == 1 && c->kind == 0)) return LIC_EINVAL;
    *sig = t->data();
    *n = (uint32_t)t->size();
    return LIC_OK;
}

// ------------------------------------------------------------------ pool
extern "C" lic_status lic_buf_acquire(lic_codec* c, size_t bytes, void** host_ptr) {
    if (!c || !host_ptr || bytes == 0) return LIC_EINVAL;
    std::lock_guard<std::mutex> g(c->pool_mu);
    auto& fl = c->free_lists[bytes];
    if (!fl.empty()) {
        *host_ptr = fl.back();
        fl.pop_back();
        ++c->pool_reuses;
        return LIC_OK;
    }
    void* p = nullptr;
    cudaSetDevice(c->device);
    if (cudaHostAlloc(&p, bytes, cudaHostAllocMapped | cudaHostAllocPortable) != cudaSuccess) {
        cudaGetLastError();
        return fail(c, LIC_ENOMEM, "cudaHostAlloc(%zu)", bytes);
    }
    c->owned[p] = bytes;
    ++c->pool_allocs;
    *host_ptr = p;
    return LIC_OK;
}

extern "C" lic_status lic_buf_release(lic_codec* c, void* host_ptr) {
    if (!c || !host_ptr) return LIC_EINVAL;
    std::lock_guard<std::mutex> g(c->pool_mu);
    auto it = c->owned.find(host_ptr);
    if (it == c->owned.end()) return LIC_EFOREIGN;
    c->free_lists[it->second].push_back(host_ptr);
    return LIC_OK;
}

extern "C" lic_status lic_buf_stats(const lic_codec* c, uint64_t* allocations, uint64_t* reuses) {
    if (!c) return LIC_EINVAL;
    std::lock_guard<std::mutex> g(const_cast<lic_codec*>(c)->pool_mu);
    if (allocations) *allocations = c->pool_allocs;
    if (reuses) *reuses = c->pool_reuses;
    return LIC_OK;
}

// ------------------------------------------------------------------ encode / decode

static OutBuf route_out(lic_codec* c, void* user, void* staging, size_t bytes) {
    void* d = c->zero_copy ? device_alias(user) : device_only(user);
    return d ? OutBuf{d, nullptr, bytes} : OutBuf{staging, user, bytes};
}
static const void* route_in(lic_codec* c, const void* user) {
    return c->zero_copy ? device_alias(user) : device_only(user);
}

static lic_status finish_out(lic_codec* c, const OutBuf& o, cudaStream_t st) {
    if (o.user) CK(cudaMemcpyAsync(o.user, o.dev, o.bytes, cudaMemcpyDeviceToHost, st));
    return LIC_OK;
}

static lic_status check_codec(lic_codec* c, uint32_t batch) {
    if (!c) return LIC_EINVAL;
    if (c->sticky) return LIC_ECUDA;
    if (batch == 0 || (int)batch > c->max_batch) return fail(c, LIC_ESHAPE, "batch %u > max_batch %d", batch, c->max_batch);
    if (cudaSetDevice(c->device) != cudaSuccess) return fail(c, LIC_ECUDA, "cudaSetDevice");
    return LIC_OK;
}

// h_s chain: z-hat (bufZ) -> y indexes (hyper decoder GPU1 and the tail of encode)
static lic_status run_hs(lic_codec* c, int B, uint8_t* idx_dev, float* dbg_sigma, cudaStream_t st) {
    lic_status r;
    if ((r = run_layer(c, c->layers[HS1], c->layers[HS1].prm, B, st))) return r;
    if ((r = run_layer(c, c->layers[HS2], c->layers[HS2].prm, B, st))) return r;
    ConvParams p = c->layers[HS3].prm;
    p.out_sym = idx_dev;
    p.out_f32 = dbg_sigma;
    return run_layer(c, c->layers[HS3], p, B, st);
}

static lic_status encode_impl(lic_codec* c, const void* frames, int hwc, uint32_t batch, int8_t* y_sym,
                              uint8_t* y_idx, int8_t* z_sym, uint64_t* n_sat, void* stream) {
    lic_status r = check_codec(c, batch);
    if (r) return r;
    if (!frames || !y_sym) return fail(c, LIC_EINVAL, "null frames / y_sym");
    const bool hyper = c->kind == 1;
    if (hyper != (y_idx != nullptr) || hyper != (z_sym != nullptr))
        return fail(c, LIC_EINVAL, "y_idx / z_sym must be given iff the codec is a hyperprior");
    cudaStream_t st = stream ? (cudaStream_t)stream : c->stream;
    const int B = (int)batch;
    const size_t fbytes = (size_t)B * 3 * c->H * c->W * (hwc ? 1 : 4);
    const void* fdev = device_only(frames);
    if (!fdev) {
        CK(cudaMemcpyAsync(c->d_frames, frames, fbytes, cudaMemcpyHostToDevice, st));
        fdev = c->d_frames;
    }
    const size_t ny = (size_t)B * c->M * (c->Hp / 16) * (c->Wp / 16);
    const size_t nz = hyper ? (size_t)B * c->N * (c->Hp / 64) * (c->Wp / 64) : 0;
    OutBuf oy = route_out(c, y_sym, c->d_ysym, ny);
    OutBuf oi = hyper ? route_out(c, y_idx, c->d_yidx, ny) : OutBuf{nullptr, nullptr, 0};
    OutBuf oz = hyper ? route_out(c, z_sym, c->d_zsym, nz) : OutBuf{nullptr, nullptr, 0};
    CK(cudaMemsetAsync(c->d_sat, 0, 8, st));
    const bool raw_ok = hwc && c->raw_tma_enabled && (3 * c->W) % 16 == 0 && ((uintptr_t)fdev & 15) == 0;
    if (raw_ok && c->l1r_ok && c->l1_int_enabled && c->l1_conv_enabled) {
        // row-halo g_a L1 (layer.h l1_rows): u8 samples by one TMA box per tile, integer MMAs
        ConvParams p = c->l1r.prm;
        p.frame = fdev; p.fr_u8 = 1; p.fr_H = c->H; p.fr_W = c->W; p.fr_top = c->top; p.fr_left = c->left;
        p.l1_int = 2;
        p.raw_tma = 1;
        CUtensorMap fmap{};
        if (!encode_u8_frame_map(&fmap, fdev, c->W, c->H, B, true))
            return fail(c, LIC_ECUDA, "cuTensorMapEncodeTiled (u8 frames) failed");
        if ((r = run_layer(c, c->l1r, p, B, st, &fmap))) return r;
    } else {
        ConvParams p = c->layers[GA1].prm;             // fused im2col: reads the frames directly
        p.frame = fdev; p.fr_u8 = hwc; p.fr_H = c->H; p.fr_W = c->W; p.fr_top = c->top; p.fr_left = c->left;
        p.l1_int = (hwc && c->l1_int_enabled) ? (c->l1_conv_enabled ? 2 : 1) : 0;
        if (p.l1_int && p.split == 2 && p.stage_bytes == 2u * 128u * 64u * 2u && c->l1_stage_split) {
            // integer u8 samples have no lo plane: the same shared memory holds twice as many
            // (hi-only) A stages, so the builders run a tile further ahead of the MMA warp
            p.stage_bytes /= 2;
            p.stages *= 2;
        }
        // u8 frames with 16-byte rows: each tile's raw patch is one TMA box of the frame
        CUtensorMap fmap{};
        p.raw_tma = 0;
        if (hwc && c->raw_tma_enabled && (3 * c->W) % 16 == 0 && ((uintptr_t)fdev & 15) == 0 &&
            encode_u8_frame_map(&fmap, fdev, c->W, c->H, B))
            p.raw_tma = 1;
        if ((r = run_layer(c, c->layers[GA1], p, B, st, p.raw_tma ? &fmap : nullptr))) return r;
    }
    for (int id : {GA2, GA3})
        if ((r = run_layer(c, c->layers[id], c->layers[id].prm, B, st))) return r;
    {
        ConvParams p = c->layers[GA4].prm;
        p.out_sym = oy.dev;
        p.sat_count = c->d_sat;
        p.out_f32 = c->debug ? c->dbg_y : nullptr;
        if ((r = run_layer(c, c->layers[GA4], p, B, st))) return r;
    }
    if (hyper) {
        if ((r = run_layer(c, c->layers[HA1], c->layers[HA1].prm, B, st))) return r;
        if ((r = run_layer(c, c->layers[HA2], c->layers[HA2].prm, B, st))) return r;
        ConvParams p = c->layers[HA3].prm;
        p.out_sym = oz.dev;
        p.sat_count = c->d_sat;
        p.out_f32 = c->debug ? c->dbg_z : nullptr;
        if ((r = run_layer(c, c->layers[HA3], p, B, st))) return r;
        if ((r = run_hs(c, B, (uint8_t*)oi.dev, c->debug ? c->dbg_s : nullptr, st))) return r;
    }
    if ((r = finish_out(c, oy, st))) return r;
    if (hyper && ((r = finish_out(c, oi, st)) || (r = finish_out(c, oz, st)))) return r;
    if (n_sat) CK(cudaMemcpyAsync(n_sat, c->d_sat, 8, cudaMemcpyDeviceToHost, st));
    if (!stream) CK(cudaStreamSynchronize(st));
    return LIC_OK;
}

extern "C" lic_status lic_encode(lic_codec* c, const float* frames, uint32_t batch, int8_t* y_sym, uint8_t* y_idx,
                                 int8_t* z_sym, uint64_t* n_sat, void* stream) {
    return encode_impl(c, frames, 0, batch, y_sym, y_idx, z_sym, n_sat, stream);
}
extern "C" lic_status lic_encode_u8(lic_codec* c, const uint8_t* frames, uint32_t batch, int8_t* y_sym,
                                    uint8_t* y_idx, int8_t* z_sym, uint64_t* n_sat, void* stream) {
    return encode_impl(c, frames, 1, batch, y_sym, y_idx, z_sym, n_sat, stream);
}

extern "C" lic_status lic_hyper_indexes(lic_codec* c, const int8_t* z_sym, uint32_t batch, uint8_t* y_idx,
                                        void* stream) {
    lic_status r = check_codec(c, batch);
    if (r) return r;
    if (c->kind != 1) return fail(c, LIC_EINVAL, "not a hyperprior codec");
    if (!z_sym || !y_idx) return fail(c, LIC_EINVAL, "null argument");
    cudaStream_t st = stream ? (cudaStream_t)stream : c->stream;
    const int B = (int)batch;
    const int Hz = c->Hp / 64, Wz = c->Wp / 64;
    const size_t nz = (size_t)B * c->N * Hz * Wz, ny = (size_t)B * c->M * (c->Hp / 16) * (c->Wp / 16);
    const int8_t* zd = (const int8_t*)route_in(c, z_sym);
    if (!zd) {
        CK(cudaMemcpyAsync(c->d_zsym, z_sym, nz, cudaMemcpyHostToDevice, st));
        zd = c->d_zsym;
    }
    OutBuf oi = route_out(c, y_idx, c->d_yidx, ny);
    CK(launch_sym_ingest(zd, c->mu_z, B, c->N, Hz, Wz, c->bufZ, c->planeZ, c->split, st));
    ++c->launches;
    if ((r = run_hs(c, B, (uint8_t*)oi.dev, nullptr, st))) return r;
    if ((r = finish_out(c, oi, st))) return r;
    if (!stream) CK(cudaStreamSynchronize(st));
    return LIC_OK;
}

static lic_status decode_impl(lic_codec* c, const int8_t* y_sym, uint32_t batch, void* frames, int u8, void* stream) {
    lic_status r = check_codec(c, batch);
    if (r) return r;
    if (!y_sym || !frames) return fail(c, LIC_EINVAL, "null argument");
    cudaStream_t st = stream ? (cudaStream_t)stream : c->stream;
    const int B = (int)batch;
    const int Hy = c->Hp / 16, Wy = c->Wp / 16;
    const size_t ny = (size_t)B * c->M * Hy * Wy;
    const int8_t* yd = (const int8_t*)route_in(c, y_sym);
    if (!yd) {
        CK(cudaMemcpyAsync(c->d_ysym, y_sym, ny, cudaMemcpyHostToDevice, st));
        yd = c->d_ysym;
    }
    const size_t fbytes = (size_t)B * 3 * c->H * c->W * (u8 ? 1 : 4);
    OutBuf of = route_frames_out(frames, c->d_frames, fbytes);
    CK(launch_sym_ingest(yd, c->kind == 0 ? c->mu_y : nullptr, B, c->M, Hy, Wy, c->bufY, c->planeY, c->split, st));
    ++c->launches;
    {
        // hyperprior y-hat = the integer symbols: exact in fp16, its lo plane is zero
        Layer& L1g = c->gs1h_ok ? c->gs1h : c->layers[GS1];
        ConvParams p1 = L1g.prm;
        p1.a_hi_only = c->kind == 1 && c->a_hi_only_enabled;
        if ((r = run_layer(c, L1g, p1, B, st))) return r;
    }
    for (int id : {GS2, GS3})
        if ((r = run_layer(c, c->layers[id], c->layers[id].prm, B, st))) return r;
    ConvParams p = c->layers[GS4].prm;
    p.out_f32 = u8 ? nullptr : (float*)of.dev;
    p.out_u8 = u8 ? (uint8_t*)of.dev : nullptr;
    if ((r = run_layer(c, c->layers[GS4], p, B, st))) return r;
    if ((r = finish_out(c, of, st))) return r;
    if (!stream) CK(cudaStreamSynchronize(st));
    return LIC_OK;
}

extern "C" lic_status lic_decode(lic_codec* c, const int8_t* y_sym, uint32_t batch, float* frames, void* stream) {
    return decode_impl(c, y_sym, batch, frames, 0, stream);
}
extern "C" lic_status lic_decode_u8(lic_codec* c, const int8_t* y_sym, uint32_t batch, uint8_t* frames,
                                    void* stream) {
    return decode_impl(c, y_sym, batch, frames, 1, stream);
}

// ------------------------------------------------------------------ test exports
static lic_status ensure_dbg(lic_codec* c) {
    if (c->d_dbg) return LIC_OK;
    lic_status r;
    const size_t ny = (size_t)c->max_batch * c->M * (c->Hp / 16) * (c->Wp / 16);
    const size_t nz = (size_t)c->max_batch * c->N * std::max(1, c->Hp / 64) * std::max(1, c->Wp / 64);
    if ((r = dalloc(c, &c->d_dbg, c->dbg_elems * 4)) || (r = dalloc(c, &c->dbg_y, ny * 4)) ||
        (r = dalloc(c, &c->dbg_z, nz * 4)) || (r = dalloc(c, &c->dbg_s, ny * 4)))
        return r;
    return LIC_OK;
}

extern "C" lic_status lic_set_debug(lic_codec* c, int on) {
    if (!c) return LIC_EINVAL;
    lic_status r = ensure_dbg(c);
    if (r) return r;
    c->debug = on;
    return LIC_OK;
}

extern "C" lic_status lic_debug_latents(lic_codec* c, uint32_t batch, float* y, float* z, float* sigma) {
    lic_status r = check_codec(c, batch);
    if (r) return r;
    if (!c->debug) return fail(c, LIC_EINVAL, "debug not enabled");
    const size_t ny = (size_t)batch * c->M * (c->Hp / 16) * (c->Wp / 16);
    const size_t nz = (size_t)batch * c->N * (c->Hp / 64) * (c->Wp / 64);
    CK(cudaStreamSynchronize(c->stream));
    if (y) CK(cudaMemcpy(y, c->dbg_y, ny * 4, cudaMemcpyDefault));
    if (c->kind == 1) {
        if (z) CK(cudaMemcpy(z, c->dbg_z, nz * 4, cudaMemcpyDefault));
        if (sigma) CK(cudaMemcpy(sigma, c->dbg_s, ny * 4, cudaMemcpyDefault));
    }
    return LIC_OK;
}

extern "C" lic_status lic_test_layer(lic_codec* c, int id, const float* in, uint32_t batch, float* out,
                                     void* stream) {
    lic_status r = check_codec(c, batch);
    if (r) return r;
    if (id < 0 || id >= NLAYER || !c->layers[id].present || !in || !out) return fail(c, LIC_EINVAL, "bad layer");
    if ((r = ensure_dbg(c))) return r;
    cudaStream_t st = stream ? (cudaStream_t)stream : c->stream;
    Layer& Ly = c->layers[id];
    const int B = (int)batch;
    const size_t nin = (size_t)B * Ly.Cin * Ly.Hin * Ly.Win;
    const size_t nout = (size_t)B * Ly.Cout * Ly.Hout * Ly.Wout;
    const float* ind = (const float*)device_only(in);
    if (!ind) {
        CK(cudaMemcpyAsync(c->d_dbg, in, nin * 4, cudaMemcpyHostToDevice, st));
        ind = c->d_dbg;
    }
    ConvParams p = Ly.prm;
    if (id == GA1) {
        // the fused L1 reads its input during the launch: keep it apart from the output scratch
        if (ind == c->d_dbg) {
            if (!c->d_dbg_in && (r = dalloc(c, &c->d_dbg_in, c->dbg_elems * 4))) return r;
            CK(cudaMemcpyAsync(c->d_dbg_in, ind, nin * 4, cudaMemcpyDeviceToDevice, st));
            ind = c->d_dbg_in;
        }
        p.frame = ind; p.fr_u8 = 0; p.fr_H = Ly.Hin; p.fr_W = Ly.Win; p.fr_top = 0; p.fr_left = 0;
    } else {
        CK(launch_pack_chw(ind, B, Ly.Cin, Ly.Hin, Ly.Win, Ly.in_buf, Ly.in_plane, c->split, st));
    }
    OutBuf o = route_out(c, out, c->d_dbg, nout * 4);
    p.out_f32 = (float*)o.dev;
    p.sat_count = nullptr;
    if (Ly.ep == EP_YQUANT || Ly.ep == EP_ZQUANT) p.out_sym = c->d_ysym;   // symbols discarded
    if (Ly.ep == EP_ZQUANT) p.out_sym = c->d_zsym;
    if (Ly.ep == EP_SIGMA) p.out_sym = c->d_yidx;
    if (Ly.ep == EP_FINAL) { p.crop_top = 0; p.crop_left = 0; p.crop_H = Ly.Hout; p.crop_W = Ly.Wout; p.out_u8 = nullptr; }
    if ((r = run_layer(c, Ly, p, B, st))) return r;
    if ((r = finish_out(c, o, st))) return r;
    if (!stream) CK(cudaStreamSynchronize(st));
    return LIC_OK;
}

extern "C" lic_status lic_test_sigma_to_index(lic_codec* c, const float* sigma, size_t n, uint8_t* idx) {
    if (!c || !sigma || !idx) return LIC_EINVAL;
    if (c->sticky) return LIC_ECUDA;
    // test-only scratch: allocated once on first use, kept until lic_close; chunks of kTestN
    constexpr size_t kTestN = (size_t)1 << 20;
    lic_status r;
    if (!c->d_test && ((r = dalloc(c, &c->d_test, kTestN * 4)) || (r = dalloc(c, &c->d_test_idx, kTestN)))) return r;
    CK(cudaSetDevice(c->device));
    for (size_t o = 0; o < n; o += kTestN) {
        const size_t m = std::min(kTestN, n - o);
        CK(cudaMemcpyAsync(c->d_test, sigma + o, m * 4, cudaMemcpyDefault, c->stream));
        CK(launch_sigma_index(c->d_test, m, c->table, c->d_test_idx, c->stream));
        CK(cudaMemcpyAsync(idx + o, c->d_test_idx, m, cudaMemcpyDefault, c->stream));
        CK(cudaStreamSynchronize(c->stream));
    }
    return LIC_OK;
}

// ------------------------------------------------------------------ measurement
extern "C" lic_status lic_profile(lic_codec* c, int on) { return lic_profile_layers(c, on ? ~0u : 0u); }

extern "C" lic_status lic_profile_layers(lic_codec* c, uint32_t mask) {
    if (!c) return LIC_EINVAL;
    const int on = mask != 0;
    c->prof_mask = mask;
    cudaSetDevice(c->device);
    if (on && c->ev.empty()) {
        c->ev.resize(2 * kProfSlots);
        c->ev_layer.resize(kProfSlots);
        for (auto& e : c->ev) CK(cudaEventCreate(&e));
    }
    if (!on) prof_flush(c);
    for (int i = 0; i < NLAYER; ++i) { c->prof_ms[i] = 0; c->prof_n[i] = 0; }
    c->ev_used = 0;
    c->profiling = on;
    return LIC_OK;
}

extern "C" lic_status lic_profile_read(lic_codec* c, int id, double* ms, uint64_t* n) {
    if (!c || id < 0 || id >= NLAYER) return LIC_EINVAL;
    cudaSetDevice(c->device);
    prof_flush(c);
    if (ms) *ms = c->prof_ms[id];
    if (n) *n = c->prof_n[id];
    return LIC_OK;
}

extern "C" lic_status lic_range_count(lic_codec* c, uint64_t* n, int reset) {
    if (!c || !n) return LIC_EINVAL;
    if (c->sticky) return LIC_ECUDA;
    CK(cudaSetDevice(c->device));
    CK(cudaDeviceSynchronize());
    unsigned long long v = 0;
    CK(cudaMemcpy(&v, c->d_range, 8, cudaMemcpyDeviceToHost));
    if (reset) CK(cudaMemset(c->d_range, 0, 8));
    *n = v;
    return LIC_OK;
}

extern "C" lic_status lic_launch_count(const lic_codec* c, uint64_t* n) {
    if (!c || !n) return LIC_EINVAL;
    *n = c->launches;
    return LIC_OK;
}

size_t lic_internal_frame_pixels(const lic_codec* c) { return c ? (size_t)c->H * c->W : 0; }

// A second codec with the same weights and geometry (own activation buffers, tensor maps and
// stream): lets a pipeline run decoder GPU1 on its own stream concurrently with the others.
lic_status lic_internal_clone(const lic_codec* c, lic_codec** out) {
    if (!c || !out) return LIC_EINVAL;
    const lic_status st = lic_open(c->licw.data(), c->licw.size(), c->device, (uint32_t)c->H, (uint32_t)c->W,
                                   (uint32_t)c->max_batch, c->precision, out);
    if (st == LIC_OK) (*out)->zero_copy = c->zero_copy;
    return st;
}

uint64_t lic_internal_launches(const lic_codec* c) { return c ? c->launches : 0; }
int lic_internal_zero_copy(const lic_codec* c) { return c ? c->zero_copy : 0; }

extern "C" lic_status lic_set_zero_copy(lic_codec* c, int on) {
    if (!c) return LIC_EINVAL;
    c->zero_copy = on ? 1 : 0;
    return LIC_OK;
}

extern "C" lic_status lic_trace(lic_codec* c, int layer_id, int on) {
    if (!c || layer_id < 0 || layer_id >= NLAYER) return LIC_EINVAL;
    if (on && !c->d_trace) {
        lic_status r = dalloc(c, &c->d_trace, 256 * kTraceEvents * 8);
        if (r) return r;
    }
    c->trace_layer = on ? layer_id : -1;
    return LIC_OK;
}

extern "C" lic_status lic_trace_read(lic_codec* c, uint64_t* out, size_t n) {
    if (!c || !out || !c->d_trace) return LIC_EINVAL;
    cudaSetDevice(c->device);
    CK(cudaStreamSynchronize(c->stream));
    CK(cudaMemcpy(out, c->d_trace, std::min<size_t>(n, 256 * kTraceEvents) * 8, cudaMemcpyDeviceToHost));
    return LIC_OK;
}
