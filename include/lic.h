/*
 * lic.h -- C ABI of the B200 learned-image-codec hot path (arXiv 2208.01641).
 *
 * The paper states the problem as "encode an image" into strings and "decode strings"
 * into an image (§III.A-B, Fig. 1); its encoder GPU workload is g_a, h_a, the
 * quantisation of z and h_s, its decoder GPU workloads are h_s (GPU1) and
 * g_s (GPU2) of the 4-stage CPU1-GPU1-CPU2-GPU2 pipeline, and the entropy
 * coder is a CPU workload.  This library therefore exports:
 *   - GPU: lic_encode      frame(s)  -> y symbols (+ y CDF indexes, z symbols)
 *          lic_hyper_indexes z symbols -> y CDF indexes         (decoder GPU1)
 *          lic_decode      y symbols -> frame(s)                (decoder GPU2)
 *   - HOST: CDF tables and the rANS coder (lic_cdf*, lic_rans_*), reentrant, no GPU.
 * Every step of the GPU path runs in this library's sm_100a kernels; there is no CPU
 * fallback.  Names follow the paper's notation (x, y, z, y-hat, z-hat, sigma).
 *
 * Conventions
 *   - Frames: f32 planar [batch][3][H][W] with values in [0,1] (lic_encode / lic_decode),
 *     or u8 interleaved [batch][H][W][3] (lic_*_u8; x = u8/255 on input, out =
 *     round_half_away(255 * x-hat) on output).  H x W is the geometry given to lic_open;
 *     the library pads it centred with zeros to a multiple of 16 (factorized) or 64
 *     (hyperprior) and crops after decode.
 *   - Symbol planes: int8 [batch][C][Hl][Wl] in channel-major raster order, values in
 *     [-L, L]; y CDF indexes uint8 with the same shape ("scales information
 *     deduced from z"; SPEC.md:135-139 SymbolPlane).  Shapes from lic_shapes.
 *   - Pointers may be device pointers, pinned host pointers (cudaHostAlloc /
 *     lic_buf_acquire: kernels read/write them in place, the paper's zero-copy,
 *     PAPER.md:84), or ordinary host pointers (staged through library-owned pinned
 *     buffers).  The caller owns every array it passes.
 *   - `stream` is a cudaStream_t passed as void*.  NULL: the library uses its own stream
 *     and returns after the work (and any host copy) is complete.  Non-NULL: work is
 *     enqueued and the call returns; outputs are valid after the caller synchronises
 *     the stream.
 *   - Device memory is allocated once in lic_open and freed only in lic_close (PAPER.md:105
 *     "we carefully control dynamic memory allocation/deallocation and pool the
 *     allocated memory"); no call allocates or frees device memory in steady state.  The
 *     batch-sized part (the workspace) may instead be owned by the caller (e.g. a torch
 *     allocation): lic_workspace_bytes / lic_bind_workspace.  Test-only exports allocate
 *     their scratch once, on first use.
 *   - Errors: every call returns lic_status; nothing aborts or throws across the ABI
 *     ("never a panic").  A CUDA failure is sticky for the codec (LIC_ECUDA).
 *   - Concurrency: one lic_codec is driven by one thread at a time; the host coder
 *     functions are reentrant and may run on any number of threads.
 */
#ifndef LIC_H
#define LIC_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct lic_codec lic_codec;

typedef enum {
    LIC_OK = 0,
    LIC_EINVAL = 1,     /* bad argument or invalid weights (beta <= 0, gamma < 0: SPEC.md:102) */
    LIC_ESHAPE = 2,     /* geometry / batch mismatch */
    LIC_ECORRUPT = 3,   /* corrupt or truncated bitstream */
    LIC_EDIGEST = 4,    /* weights container failed validation */
    LIC_ENOMEM = 5,     /* allocation failed (only in lic_open / pool growth) */
    LIC_ECUDA = 6,      /* CUDA error (sticky) or no sm_100 device */
    LIC_EFOREIGN = 7,   /* buffer not owned by this pool */
    LIC_ENOSPACE = 8    /* output capacity too small */
} lic_status;

typedef struct { uint32_t c, h, w; } lic_shape;

typedef enum {
    LIC_PREC_SPLIT = 0, /* activations as fp16 hi + lo planes, fp32 accumulation (graded) */
    LIC_PREC_F16 = 1    /* single fp16 activation plane (the paper's TensorRT FP16) */
} lic_precision;

/* ---------------------------------------------------------------- codec lifetime */

/* Parse and validate an LICW weights container (layout in DESIGN.md §4),
 * upload the weights to `device`, plan every layer for frames of height x width and up
 * to max_batch frames per call, allocate all device memory.  `licw` is only read during
 * the call.  Errors: LIC_EDIGEST (malformed container), LIC_EINVAL (beta <= 0, gamma < 0,
 * unsupported N/M, or a conv / deconv weight or gamma entry that is not exactly
 * representable in fp16 -- the tensor cores take fp16 operands and the split-FP16 mode
 * (R16) is exact only for fp16 weights, as the paper's FP16 engines hold them,
 * PAPER.md:129; round trained weights to fp16 once, then run the oracle on the same
 * rounded values), LIC_ESHAPE (zero geometry), LIC_ECUDA (no sm_100 device), LIC_ENOMEM.
 * On failure *out is NULL and lic_last_error(NULL) returns this thread's message. */
lic_status lic_open(const uint8_t* licw, size_t len, int device, uint32_t height, uint32_t width,
                    uint32_t max_batch, int precision, lic_codec** out);
void lic_close(lic_codec* codec);

/* Latent shapes per frame: y = M x Hp/16 x Wp/16; z = N x Hp/64 x Wp/64 (z = {0,0,0}
 * for the factorized codec).  `kind` receives 0 (factorized) or 1 (hyperprior). */
lic_status lic_shapes(const lic_codec* codec, lic_shape* y, lic_shape* z, int* kind);

/* Zero-copy toggle ("we offer a command-line option ... to quickly toggle
 * this option on or off").  Off (default): host symbol planes move by DMA through
 * device staging buffers.  On: kernels read/write pinned host planes in place over PCIe
 * (the paper's unified-memory Jetson path). */
lic_status lic_set_zero_copy(lic_codec* codec, int on);

/* Message for the last error on this codec (owned by the codec); codec == NULL: the last
 * failed lic_open on the calling thread (thread-local). */
const char* lic_last_error(const lic_codec* codec);

/* ---------------------------------------------------------------- workspace
 * device memory is allocated once and pooled, never freed while the codec
 * runs.  The batch-sized device memory of a codec -- activation planes (fp16 hi + lo NHWC
 * ping-pong buffers of the largest activation, the y- and z-planes), frame staging and
 * symbol / index staging planes -- is one block, "the workspace".  lic_open allocates it
 * for max_batch frames; a caller that owns device memory (PyTorch's caching allocator)
 * may hand the codec its own block instead.
 *
 * lic_workspace_bytes: bytes of the workspace for `batch` frames (0: lic_open's
 *   max_batch); 0 if batch exceeds it or codec is NULL.
 * lic_bind_workspace: waits for the device, then uses [dev_ptr, dev_ptr + bytes) as the
 *   workspace from now on and frees the library's own block.  The codec's max_batch
 *   becomes the largest batch (<= lic_open's) whose workspace fits in `bytes`
 *   (lic_max_batch).  dev_ptr must be device memory of the codec's device, 256-byte
 *   aligned; the caller keeps it alive until lic_close or the next bind.  Results are
 *   bit-identical to the library-owned workspace.  Errors: LIC_EINVAL (NULL, host memory,
 *   wrong device, misaligned), LIC_ENOSPACE (smaller than one frame's workspace). */
size_t lic_workspace_bytes(const lic_codec* codec, uint32_t batch);
lic_status lic_bind_workspace(lic_codec* codec, void* dev_ptr, size_t bytes);
lic_status lic_max_batch(const lic_codec* codec, uint32_t* max_batch);

/* ---------------------------------------------------------------- pooled pinned buffers */

/* Pinned, device-mapped host buffers from an exact-size free-list pool (
 * PAPER.md:84 zero-copy, :105 pooling).  Kernels write symbol planes straight into them.
 * acquire reuses a released buffer of the same size before allocating.  release of a
 * pointer not from this pool returns LIC_EFOREIGN. */
lic_status lic_buf_acquire(lic_codec* codec, size_t bytes, void** host_ptr);
lic_status lic_buf_release(lic_codec* codec, void* host_ptr);
/* counters: allocations, reuses (SPEC.md:359 pool_allocations / pool_reuses) */
lic_status lic_buf_stats(const lic_codec* codec, uint64_t* allocations, uint64_t* reuses);

/* ---------------------------------------------------------------- GPU entry points */

/* Encode (PAPER.md:68 factorized, :74 hyperprior GPU workload):
 *   x -> g_a -> y; factorized: y_sym = clamp(round_half_away(y - mu_c), -L, L);
 *   hyperprior: z = h_a(|y|), z_sym = clamp(round(z - mu_z)), z-hat = z_sym + mu_z,
 *   sigma = h_s(z-hat), y_idx = #{j <= 62 : table_j < max(sigma, 0.11)},
 *   y_sym = clamp(round(y)).
 * y_idx and z_sym must be NULL for the factorized codec and non-NULL for the hyperprior.
 * n_saturated (nullable) receives the number of clamped symbols.  batch <= max_batch. */
lic_status lic_encode(lic_codec* codec, const float* frames, uint32_t batch,
                      int8_t* y_sym, uint8_t* y_idx, int8_t* z_sym, uint64_t* n_saturated,
                      void* stream);
lic_status lic_encode_u8(lic_codec* codec, const uint8_t* frames_hwc, uint32_t batch,
                         int8_t* y_sym, uint8_t* y_idx, int8_t* z_sym, uint64_t* n_saturated,
                         void* stream);

/* Hyperprior decoder stage GPU1: z_sym -> z-hat -> h_s -> y CDF indexes.
 * Bit-identical to the y_idx lic_encode produced from the same z symbols. */
lic_status lic_hyper_indexes(lic_codec* codec, const int8_t* z_sym, uint32_t batch,
                             uint8_t* y_idx, void* stream);

/* Decoder stage GPU2: y-hat = y_sym + mu_c (hyperprior: mu = 0),
 * x-hat = clamp(g_s(y-hat), 0, 1) cropped to H x W. */
lic_status lic_decode(lic_codec* codec, const int8_t* y_sym, uint32_t batch, float* frames,
                      void* stream);
lic_status lic_decode_u8(lic_codec* codec, const int8_t* y_sym, uint32_t batch,
                         uint8_t* frames_hwc, void* stream);

/* ---------------------------------------------------------------- test-only exports
 * Same device code as the hot path, exposed for per-layer parity tests. */

/* Layer ids: 0-3 g_a L1-L4, 4-7 g_s L1-L4, 8-10 h_a L1-L3, 11-13 h_s L1-L3.
 * in: f32 [batch][Cin][Hin][Win] (the layer's input in padded coordinates; for g_a L1 the
 * padded frame); out: f32 [batch][Cout][Hout][Wout] = the layer's output after its fused
 * activation (g_a L4: y; h_a L3: z; h_s L3: sigma after ReLU; g_s L4: clamp to [0,1]). */
lic_status lic_test_layer(lic_codec* codec, int layer_id, const float* in, uint32_t batch,
                          float* out, void* stream);
/* Shapes of a layer: input (c,h,w) and output (c,h,w). */
lic_status lic_layer_shapes(const lic_codec* codec, int layer_id, lic_shape* in, lic_shape* out);
/* sigma -> index exactly as the h_s L3 epilogue computes it, on a given sigma array. */
lic_status lic_test_sigma_to_index(lic_codec* codec, const float* sigma, size_t n, uint8_t* idx);
/* When enabled, lic_encode also keeps y (and z, sigma) as f32 for lic_debug_latents. */
lic_status lic_set_debug(lic_codec* codec, int on);
lic_status lic_debug_latents(lic_codec* codec, uint32_t batch, float* y, float* z, float* sigma);

/* ---------------------------------------------------------------- measurement
 * When profiling is on, every GEMM-engine launch is bracketed by CUDA events recorded on
 * the stream it is launched on; lic_profile_read synchronises and returns the summed
 * device time and launch count per layer since profiling was enabled (then resets). */
lic_status lic_profile(lic_codec* codec, int on);
/* The same for a subset of layers: bit i of `mask` = layer id i (0: off).  Events between
 * kernels serialise them, so a timed run brackets only the layers it reports. */
lic_status lic_profile_layers(lic_codec* codec, uint32_t mask);
lic_status lic_profile_read(lic_codec* codec, int layer_id, double* ms, uint64_t* launches);
/* Test-only timeline: while on, launches of `layer_id` record clock64 events of CTA 0 per
 * tile (MMA start/end, norm issue, epilogue start / x^2 written / norm ready / end, producer
 * start, builder / MMA-issue points); lic_trace_read copies up to n values (256 tiles x 24 slots). */
lic_status lic_trace(lic_codec* codec, int layer_id, int on);
lic_status lic_trace_read(lic_codec* codec, uint64_t* out, size_t n);
/* Total kernels this codec has launched (GEMM engine + ingest kernels). */
lic_status lic_launch_count(const lic_codec* codec, uint64_t* n);

/* Activation range guard (R16d).  Activations are stored as fp16 hi + lo planes
 * whose range ends at 65504 -- the bound of the paper's FP16 engines.  (The
 * GDN / IGDN norm operand x^2 is scaled per pixel by an exact power of two, so it has no
 * such bound.)  An activation beyond +-65504 is stored saturated to +-65504 -- never inf
 * or NaN -- and counted; a nonzero count means the results of the calls since the last
 * reset may differ from the fp32 oracle.  Waits for the device (a diagnostic, not a
 * hot-path call); *n = the count since the last reset; reset != 0 zeroes it. */
lic_status lic_range_count(lic_codec* codec, uint64_t* n, int reset);

/* ---------------------------------------------------------------- HOST entropy coder */

/* CDF tables of this codec: which = 0 factorized y rows (one per
 * channel, from sigma_c), 1 z rows (one per channel, sigma_z), 2 Gaussian rows (one per
 * scale-table entry).  Rows are row_len = 2L+2 uint32 cumulative frequencies 0..65536.
 * The table is owned by the codec.  LIC_EINVAL if the codec has no such table. */
lic_status lic_cdf(const lic_codec* codec, int which, const uint32_t** rows, uint32_t* n_rows,
                   uint32_t* row_len);

/* The scales those tables are built from: which = 0 sigma_y (factorized, one per y channel),
 * 1 sigma_z (hyperprior, one per z channel), 2 the 64-entry scale table (hyperprior y rows).
 * Pointer valid while the codec lives.  LIC_EINVAL if the codec has no such table. */
lic_status lic_sigmas(const lic_codec* codec, int which, const float** sigmas, uint32_t* n);

/* Build one CDF row per sigma (zero-mean discretised Gaussian over [-L, L], tails folded,
 * 16-bit quantised, every frequency >= 1).  out: n x (2L+2) uint32. */
lic_status lic_cdf_build(const float* sigmas, uint32_t n, uint32_t L, uint32_t* out);

/* rANS: 32-bit state, L = 2^23, byte-wise
 * renormalisation, 16-bit precision, symbols coded in reverse raster order, 4-byte
 * big-endian final state at the front.  Symbol s uses CDF row `row[i]` (uint8, per symbol)
 * or, if row == NULL, row = channel index of the C x H x W plane.  Symbol s occupies CDF
 * entries [s - sym_min, s - sym_min + 1].  out: capacity `cap` bytes, written length in
 * *out_len.  Errors: LIC_EINVAL (symbol out of range / bad row), LIC_ENOSPACE (cap). */
lic_status lic_rans_encode(const int8_t* sym, const uint8_t* row, lic_shape plane,
                           const uint32_t* cdf, uint32_t n_rows, uint32_t row_len, int sym_min,
                           uint8_t* out, size_t cap, size_t* out_len);
/* Inverse of lic_rans_encode.  LIC_ECORRUPT if the stream is exhausted early, a slot is
 * outside the table, or the final state is not 2^23 with every byte consumed. */
lic_status lic_rans_decode(const uint8_t* in, size_t len, const uint8_t* row, lic_shape plane,
                           const uint32_t* cdf, uint32_t n_rows, uint32_t row_len, int sym_min,
                           int8_t* sym_out);

/* ---------------------------------------------------------------- streaming pipeline
 * The paper's architecture (§III.A-B, Fig. 2): every frame is a task that moves
 * through GPU and CPU workloads; one dedicated control thread drives the GPU (encode,
 * decoder GPU1 = lic_hyper_indexes, decoder GPU2 = lic_decode) and a pool of worker
 * threads runs the rANS coder (encode y/z, decode z, decode y).  Batches of frames are
 * double-buffered in pooled pinned slots so that no GPU work waits on the host coder and
 * vice versa.  lic_pipeline_run pushes `nframes` frames through the full round trip
 * encode -> bitstreams -> decode.  serial = 1 runs the serial reference instead (each
 * batch completes every stage before the next starts). */
typedef struct lic_pipeline lic_pipeline;
typedef struct {
    uint32_t coder_threads;   /* host coder workers (the paper uses 3 and 10: PAPER.md:155, :163) */
    uint32_t batch;           /* frames per GPU call (<= codec max_batch) */
    uint32_t inflight;        /* batches in flight (>= 2 double-buffers) */
    int u8;                   /* frames are u8 [H][W][3] (1) or f32 [3][H][W] (0) */
    int serial;               /* 1: no overlap between stages (reference) */
    int keep_bitstreams;      /* 1: keep every frame's strings for lic_pipeline_bitstream */
    uint32_t substreams;      /* y string as K channel-slab substreams (lic_rans_encode_slabs); 0 or 1: one string */
    uint32_t coder;           /* 0: 32-bit rANS over the codec's +-L tables (above); 1: rans64 + bypass escape
                                 (lic_rans64_*, R23) with Gaussian tables (tail 1e-9) on the
                                 codec's scales (lic_sigmas); one string per plane, substreams ignored */
    float pace_fps;           /* > 0: paced source -- batch i is submitted at t0 + i * batch / pace_fps and its
                                 latency counts from that submission (queueing included);
                                 0: every frame is available at the start, latency counts from the
                                 batch's admission into a slot */
    uint32_t timeline;        /* 1: record lic_pipeline_timeline events for the run */
    uint32_t coder_parts;     /* hyperprior, coder 0, substreams K: each frame's y string is coded (and decoded) as
                                 this many slab ranges on separate coder threads (lic_rans_encode_slab_range) --
                                 the same bitstream, 1/parts of the per-frame coder latency; 0 or 1: one task */
} lic_pipeline_config;
typedef struct {
    uint64_t frames;          /* frames completed */
    double seconds;           /* wall time of the run */
    double latency_p50_ms, latency_p95_ms, latency_max_ms; /* per batch: submission (paced) or slot admission
                                                              (unpaced) -> decode complete */
    uint64_t y_bytes, z_bytes;/* total bitstream bytes */
    uint64_t symbol_mismatches; /* decoded != encoded symbols (must be 0: lossless) */
    double gpu_busy_s, coder_busy_s; /* summed busy time of the GPU thread / coder threads */
    uint64_t gpu_launches;    /* kernels launched by the run (all of the pipeline's codecs) */
} lic_pipeline_stats;
lic_status lic_pipeline_open(lic_codec* codec, const lic_pipeline_config* cfg, lic_pipeline** out);
void lic_pipeline_close(lic_pipeline* p);
/* frames_in / frames_out: nframes frames, device or pinned-host pointers (zero-copy).
 * nframes must be a multiple of cfg->batch. */
lic_status lic_pipeline_run(lic_pipeline* p, const void* frames_in, uint32_t nframes, void* frames_out,
                            lic_pipeline_stats* stats);
/* Timeline of the last run (cfg.timeline = 1), the evidence for the overlap the paper's
 * architecture is built on ("the GPU and CPU workloads ... are executed
 * concurrently").  One record per GPU task (kind 0 encode, 1 decoder GPU1, 2 decoder GPU2;
 * lane = the stream: 0 main, 1 GPU1's own stream; start / end = device time of the task's
 * first / last kernel from CUDA events) and per coder task (kind 3 = E(y), E(z) and decoder
 * CPU1, kind 4 = decoder CPU2; lane = worker thread; host clock).  t_ready = when the task
 * could have started (slot free / submitted, or its inputs decoded).  Times in ms since the
 * run started.  *n = the number of records; LIC_ENOSPACE if cap is smaller (out holds cap). */
typedef struct {
    uint32_t kind, lane;
    int32_t batch, frame;     /* frame within the batch; -1 for GPU tasks */
    double t_ready_ms, t_start_ms, t_end_ms;
} lic_timeline_event;
lic_status lic_pipeline_timeline(const lic_pipeline* p, lic_timeline_event* out, size_t cap, size_t* n);
/* strings of frame i of the last run (keep_bitstreams = 1); z is NULL/0 for factorized. */
lic_status lic_pipeline_bitstream(const lic_pipeline* p, uint32_t frame, const uint8_t** y, size_t* y_len,
                                  const uint8_t** z, size_t* z_len);

/* Prepared coder tables (same bitstream as lic_rans_encode / lic_rans_decode, faster):
 * per (row, symbol) encoder constants with an exact reciprocal in place of the division
 * x / freq, and a 4096-bucket slot -> symbol index per row for the decoder.  Immutable
 * after lic_rans_prepare; shareable across threads.  `cdf` is copied. */
typedef struct lic_rans_tables lic_rans_tables;
lic_status lic_rans_prepare(const uint32_t* cdf, uint32_t n_rows, uint32_t row_len, int sym_min,
                            lic_rans_tables** out);
void lic_rans_tables_free(lic_rans_tables* t);
lic_status lic_rans_encode_fast(const lic_rans_tables* t, const int8_t* sym, const uint8_t* row, lic_shape plane,
                                uint8_t* out, size_t cap, size_t* out_len);
lic_status lic_rans_decode_fast(const lic_rans_tables* t, const uint8_t* in, size_t len, const uint8_t* row,
                                lic_shape plane, int8_t* sym_out);

/* Channel-slab substreams ("the entropy coding process
 * is highly CPU-intensive", :195 faster coders as future work; reading R21).  The
 * C x H x W plane is cut into K channel slabs, slab k = channels [floor(k*C/K),
 * floor((k+1)*C/K)), and every slab is coded as an independent string in exactly the
 * lic_rans_encode format (rows as there: row[i] per symbol, or the channel).
 *   K == 1: the plain string (identical to lic_rans_encode_fast).
 *   K >  1: K big-endian u32 string lengths, then the K strings in slab order.
 * One call codes the K strings in lockstep on the calling thread (independent dependency
 * chains overlap in the core).  1 <= K <= min(64, C).  Errors as lic_rans_encode /
 * lic_rans_decode; a framing whose lengths do not add up to `len` is LIC_ECORRUPT. */
lic_status lic_rans_encode_slabs(const lic_rans_tables* t, const int8_t* sym, const uint8_t* row, lic_shape plane,
                                 uint32_t K, uint8_t* out, size_t cap, size_t* out_len);
lic_status lic_rans_decode_slabs(const lic_rans_tables* t, const uint8_t* in, size_t len, const uint8_t* row,
                                 lic_shape plane, uint32_t K, int8_t* sym_out);
/* The same coder split across threads: slabs [k_begin, k_end) of the K-slab plane only.
 * encode: the range's strings back to back in `out` (no header), their lengths in
 * lens[0 .. k_end-k_begin); a caller that concatenates the ranges of 0..K in order behind the
 * K big-endian lengths has exactly lic_rans_encode_slabs' stream.  decode: `in` is the whole
 * framed stream (header + K strings); only the range's channels of sym_out are written.
 * sym / row / sym_out are whole-plane arrays.  Errors as lic_rans_encode_slabs /
 * lic_rans_decode_slabs; LIC_EINVAL for an empty or out-of-range slab range. */
lic_status lic_rans_encode_slab_range(const lic_rans_tables* t, const int8_t* sym, const uint8_t* row, lic_shape plane,
                                      uint32_t K, uint32_t k_begin, uint32_t k_end, uint8_t* out, size_t cap,
                                      uint32_t* lens, size_t* out_len);
lic_status lic_rans_decode_slab_range(const lic_rans_tables* t, const uint8_t* in, size_t len, const uint8_t* row,
                                      lic_shape plane, uint32_t K, uint32_t k_begin, uint32_t k_end, int8_t* sym_out);

/* ---------------------------------------------------------------- rans64 + bypass escape
 * the coder the paper's implementations link ("simply integrate
 * the CompressAI entropy coder [8]") -- 64-bit rANS (L = 2^31, 32-bit words,
 * precision 16) with escape coding of values outside a table's support, R23.
 * Host only, reentrant.  Tables: n_cdfs rows of `stride` uint32 (row r valid on
 * [0, sizes[r]), c[0] = 0, c[sizes[r]-1] = 65536, strictly increasing, 3 <= sizes[r] <=
 * stride); symbol value s of row r codes v = s - offsets[r]; v outside [0, sizes[r]-2) is
 * sent as the escape (entry sizes[r]-2) plus its 4-bit "bypass" chunks, so every int32 is
 * codable.  Stream: little-endian u32 words, final state (low, high) first. */

/* Quantised CDF of pmf[0..n) (the last entry is the escape's tail mass): n + 1 entries into
 * cdf; each frequency >= 1, total 65536.  LIC_EINVAL: negative / non-finite / all-zero pmf. */
lic_status lic_cdf_quantize(const float* pmf, uint32_t n, uint32_t* cdf);
/* Gaussian tables for scales[0..n) with total tail mass `tail_mass` (CompressAI's
 * GaussianConditional construction, fp64): row r covers |k| <= center_r = ceil(scale_r *
 * m), Phi(-m) = tail_mass / 2, offsets[r] = -center_r, sizes[r] = 2 center_r + 3.
 * LIC_ENOSPACE if a row needs more than `stride` entries. */
lic_status lic_cdf64_gaussian(const float* scales, uint32_t n, double tail_mass, uint32_t* cdfs,
                              uint32_t stride, int32_t* sizes, int32_t* offsets);
/* Encode sym[0..n) with rows idx[0..n) into out (capacity cap; written length in *out_len,
 * a multiple of 4).  LIC_EINVAL: bad table / row index; LIC_ENOSPACE: cap too small
 * (8 + 8n bytes always suffice). */
lic_status lic_rans64_encode(const int32_t* sym, const int32_t* idx, size_t n, const uint32_t* cdfs,
                             uint32_t n_cdfs, uint32_t stride, const int32_t* sizes, const int32_t* offsets,
                             uint8_t* out, size_t cap, size_t* out_len);
/* Inverse of lic_rans64_encode.  LIC_ECORRUPT if the words run out, an escape is longer than
 * 9 chunks or its value leaves int32, or the final state is not 2^31 with every word read. */
lic_status lic_rans64_decode(const uint8_t* in, size_t len, const int32_t* idx, size_t n, const uint32_t* cdfs,
                             uint32_t n_cdfs, uint32_t stride, const int32_t* sizes, const int32_t* offsets,
                             int32_t* sym_out);

/* Library version string. */
const char* lic_version(void);

#ifdef __cplusplus
}
#endif
#endif /* LIC_H */
