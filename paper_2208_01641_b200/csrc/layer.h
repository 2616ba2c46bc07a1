// layer.h -- host/device description of one implicit-GEMM layer launch.
//
// Every transform layer of the codec (Fig. 1: g_a, g_s, h_a, h_s; layer shapes
// SPEC.md:319) runs through ONE persistent tcgen05 kernel (conv_umma.cu).  A layer is
//   D[pixel, co] = sum_{tap, ci} A[pixel shifted by tap, ci] * W[tap][co][ci]
// over a GEMM grid of output pixels (conv) or of input pixels per sub-pixel phase
// (stride-2 transposed conv, 4 phases with 9/6/6/4 taps), followed by a fused epilogue
// (GDN / IGDN / ReLU / quantise / sigma->index / clamp+crop).
#pragma once
#include <cstddef>
#include <cstdint>

namespace lic {

enum EpKind : int {
    EP_F32 = 0,     // acc + bias -> f32 CHW (test export)
    EP_GDN = 1,     // GDN  (x / sqrt(beta + gamma x^2))  -> fp16 hi/lo NHWC
    EP_IGDN = 2,    // IGDN (x * sqrt(beta + gamma x^2))  -> fp16 hi/lo NHWC
    EP_RELU = 3,    // max(x, 0)                          -> fp16 hi/lo NHWC
    EP_YQUANT = 4,  // s = clamp(round(y - mu)) -> int8 CHW; optional |y| -> hi/lo NHWC
    EP_ZQUANT = 5,  // s = clamp(round(z - mu)) -> int8 CHW; z-hat = s + mu -> hi/lo NHWC
    EP_SIGMA = 6,   // sigma = relu(x); idx = #{table_j < max(sigma, 0.11f)} -> uint8 CHW
    EP_FINAL = 7,   // clamp(x, 0, 1), crop -> f32 CHW and/or u8 HWC
    EP_PARTIAL = 8, // split-K: the raw fp32 accumulator of one K slice -> part[split] NHWC (summed by
                    // split_reduce_kernel, which applies the layer's own epilogue)
};

constexpr int kMaxTaps = 32;
constexpr int kMaxTps = 4;      // halo mode: at most 4 taps per weight stage
constexpr int kTraceEvents = 24; // test-only per-tile timeline slots (lic_trace_read: 256 tiles x 24)
constexpr int kBM = 128;        // pixels per tile (UMMA M)
constexpr int kBK = 64;         // channels per K chunk (one 128-byte swizzle row of fp16)

struct ConvParams {
    // ---- GEMM geometry
    int batch;
    int Cin, kchunks;                 // Cin multiple of 64
    int Cout, BN, n_ntiles;           // real output channels, N tile, #N tiles
    int Hg, Wg;                       // GEMM grid (conv: output; deconv: input grid, per phase)
    int Wt, Ht, tiles_x, tiles_y;     // tile = Ht x Wt pixels, Wt * Ht = 128
    int nphase;                       // 1 conv, 4 deconv
    int stride;                       // A coordinate = stride * g + tap offset
    int out_s;                        // output pixel = out_s * g + phase offset
    int ntaps[4], tap0[4];
    int tap_dy[kMaxTaps], tap_dx[kMaxTaps], tap_w[kMaxTaps];
    uint32_t tapoff[kMaxTaps];        // halo mode: tap t's window start in the halo, 16-byte descriptor units
                                      // ((dy + 1) * halo_w + dx + 1) * 8 -- host-computed (uniform operands)
    int split;                        // 2: activations are fp16 hi + lo planes; 1: hi only
    int cg;                           // 1: one CTA per tile; 2: CTA pair (cta_group::2, M = 256)
    int total_tiles;
    // tile-index decode without hardware division: q = (umulhi(n, m) + n) >> s (host-computed
    // magic numbers, exact for n < 2^31); Wt and nphase are powers of two
    uint32_t fd_nt_m, fd_txs_m, fd_ty_m;
    int fd_nt_s, fd_txs_s, fd_ty_s;
    int txs, wt_log2, nph_log2;
    // ---- kernel resources (host-computed)
    int stages;
    uint32_t stage_bytes, off_gamma, off_bar, off_par, smem_bytes;
    // halo mode (stride-1 layers: 3x3 convs, sub-pixel deconv phases, packed g_s L4):
    // per 64-channel chunk the (Ht+2) x (Wt+2) input halo (hi + lo) is loaded once into a
    // 2-slot ring and every tap reads its A operand as a shifted window of it; the stage
    // ring then carries only weight tiles.  Tile fixed at Wt = 8, Ht = 16.
    int halo, halo_slots, halo_w;      // halo_w: halo row pitch in pixels (>= Wt + 2)
    int tps;                          // halo mode: taps per weight stage (1 .. kMaxTps)
    int sub4;                         // halo mode for a 5x5/s2 conv: 4 parity sub-grid halos per chunk,
                                      // tap groups tap0[g] / ntaps[g] (g = py * 2 + px)
    uint32_t off_halo, halo_plane_bytes;
    int halo_planes;                  // planes per halo ring slot: split, or 1 for a plan whose input is hi-only
    int wres;                         // all weight tiles resident in smem (loaded once per CTA)
    uint32_t off_wres;
    int tmem_cols, acc_stride, n_accbuf;
    // ---- epilogue
    int ep;
    int Hout, Wout;                   // output tensor spatial size (padded coordinates)
    const float* bias;                // [Cout]
    const float* beta;                // [Cout] (GDN/IGDN)
    const float* mu;                  // [Cout] quantisation offsets, nullable (= 0)
    const float* table;               // [64] scale table (EP_SIGMA)
    int L;                            // symbol support bound
    void* out_act;                    // fp16 [split][batch][Hout][Wout][Cout]
    size_t act_plane;                 // elements per plane of out_act
    void* out_sym;                    // int8 / uint8 [batch][Cout][Hout][Wout]
    float* out_f32;                   // f32 [batch][Cout][Hout or crop_H][Wout or crop_W]
    uint8_t* out_u8;                  // u8 [batch][crop_H][crop_W][3]
    int abs_out;                      // EP_YQUANT: also write |y| planes
    int onedn;                        // EP_GDN / EP_IGDN as 1DN: the norm
                                      // contracts |x| (not x^2) with gamma and y = x / n (x * n inverse)
    int pack4;                        // EP_FINAL of a stride-2 deconv with all 4 sub-pixel
                                      // phases packed into N: column j = phase (j>>2), channel (j&3)
    int crop_top, crop_left, crop_H, crop_W;
    unsigned long long* sat_count;    // saturation counter (nullable)
    unsigned long long* range_count;  // activations outside the fp16 range (|x| > 65504), stored
                                      // saturated to +-65504 (nullable; R16d)
    unsigned long long* trace;        // test-only: per-tile clock64 events of CTA 0 (nullable)
    int dbg_nostore;                  // test-only experiment switch: skip activation stores
    int pdl;                          // launched with programmatic stream serialization: constants and
                                      // the prologue overlap the previous kernel; griddepcontrol.wait
                                      // before any global read of its outputs or any global write
    // fused g_a L1 (im2col GEMM, K = 75 padded to 128): warps 0, 2 and 3 build the A tiles
    // (hi, lo) in shared memory straight from the frame -- u8 HWC (x = u8 / 255) or f32 CHW --
    // through a per-tile input patch; no ingest kernel and no im2col tensor in HBM.  Tile fixed
    // at Wt = 16, Ht = 8 (patch 19 rows x 35 px x 3 ch fp32, double-buffered); stage s holds K
    // chunk s; the weights stay resident.
    int fuse_l1;
    const void* frame;                // u8 [B][H][W][3] or f32 [B][3][H][W] (device)
    int fr_u8, fr_H, fr_W, fr_top, fr_left;   // frame size and its offset in the padded grid
    int a_hi_only;                    // the input activation is exact in fp16 (lo plane zero: the hyperprior's
                                      // integer y-hat into g_s L1): no lo loads, no lo MMAs
    int l1_int;                       // u8 frames: A holds the integer sample (exact in fp16) -- one MMA pass,
                                      // no lo plane -- and the epilogue scales the sum by 1/255; 2: the
                                      // builders convert u8 -> f16 arithmetically (no LUT)
    uint32_t off_patch;               // split patch [2][hi, lo][19][112] fp16
    uint32_t off_lut;                 // u8 LUT [257] (hi | lo << 16; entry 256 = 0)
    uint32_t off_raw;                 // raw u8 patch [2][19][112] in 2176-byte slots (cp.async or TMA, u8 frames)
    int raw_tma;                      // the raw patch by one TMA box per tile (mapA = the u8 frame, 3W x H x B)
    // row-halo g_a L1 (u8 frames, raw TMA, integer samples; tile Wt = 8 x Ht = 16): instead of an
    // im2col A tile (128 px x 80 K) the builders write one "row halo" per tile -- element
    // (iy, tx), iy < 35, tx < 8, holds the 16 u8 samples at input row iy, bytes 6 tx .. 6 tx + 15
    // of the patch (the 5 kx taps x 3 channels of K row ky, slot 15 has a zero weight) -- and the
    // 5 kernel rows ky are 5 K = 16 MMAs whose A operand is the window of rows 2 ty + ky
    // (SW128 rows, window start ky x 1024 B, 8-row-group stride 2048 B): 2.3x fewer builder
    // stores than im2col, no fp16 patch, 5 instead of 8 MMAs per tile
    int l1_rows;
    int no_guard;                     // forward GDN / 1DN with a provable |y| bound below the fp16 range
                                      // (host check of gamma, beta; R16f): no range guard in P2
    // TMA-store epilogue: each epilogue warp stages 32 px x 16 ch (hi, lo: 1 KB each) in smem and
    // writes it with a bulk tensor store; out maps: conv (C, W, H, B), deconv phase view
    // (C, px, W/2, py, B*H/2) of the NHWC output, one map per plane
    int tma_out, ostage_slots;        // staging buffers per warp (1 or 2, 2 KB each)
    uint32_t off_ostage;
    // GDN / IGDN layers with 64 KB of staging: every epilogue warp stages its own 32 pixels in
    // rounds of wst_ch channels (32: 4 KB slots, 64-byte rows; 16: 2 KB) in wst_slots private
    // slots and stores them itself (out maps with a wst_ch-channel box); 0: quadrant blocks
    int wst_ch, wst_slots;
    // two-group GDN / IGDN epilogue (BN = 128, per-warp 32-channel staging, double-buffered TMEM):
    // two groups of 8 epilogue warps alternate tiles so one group's norm MMA round trip overlaps
    // the other's arithmetic; y is computed from the norm operand and the signs (conv_umma.cu)
    int g2;
    // split-K (few-tile h layers): tile t of the launch is (output tile t / ksplit, K slice t % ksplit);
    // slice s runs the flattened (chunk, parity group, tap) range [s U / ksplit, (s + 1) U / ksplit)
    int ksplit;
    int ksplit_ok;                    // host: the layer may be split (run_layer picks ksplit from the batch)
    float* part;                      // EP_PARTIAL: fp32 [ksplit][batch][Hout][Wout][Cout]
    int mma_spin;                     // g2: the MMA warp polls its operand barriers (test_wait loop) instead
                                      // of a suspending try_wait
    // gather mode (g_s L4, stride-2 transposed conv N -> 3): the 9 input offsets go into N instead
    // of K -- P[p][t][j] = A[p] . W_t[j] over a 16 x 8 input tile (one A read per pixel, N = 9 x 16),
    // then out[g][j] = sum_t P[g + off_t][t][j] gathered through shared memory for the 14 x 6
    // interior; tiles step by (tsx, tsy) = (14, 6) and start one pixel up-left (TMA zero fill)
    int gather;
    int tsx, tsy;                     // tile step (= Wt, Ht except in gather mode)
    uint32_t off_gp;                  // P staging: [9][128 px][12] f32
};

}  // namespace lic
