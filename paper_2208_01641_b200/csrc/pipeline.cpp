// pipeline.cpp -- the streaming runtime: GPU workloads and the host entropy coder overlapped.
//
// PAPER.md §III.A: "Each frame ... is represented by a state-machine pattern task, which
// must be processed by the above workloads sequentially.  For each workload, a FIFO task
// queue implementing a multi-threaded producer-consumer pattern manages the execution of
// the tasks ... for a GPU-intensive workload, a dedicated control thread fetches the tasks
// and communicate with the GPU; for a CPU-intensive workload, multiple worker threads
// perform the computations."  §III.B: the hyperprior encoder is 2-stage (GPU: g_a, h_a,
// Q(z), h_s; CPU: Q(y), E(y), E(z)) and the decoder 4-stage (CPU1 E^-1(z), GPU1 h_s,
// CPU2 E^-1(y), GPU2 g_s).  §III.D: memory is pooled, never freed in steady state.
//
// B200 design: the calling thread is the GPU control thread; it services three GPU task
// kinds (ENC, IDX = decoder GPU1, DEC = decoder GPU2) from a ready queue, oldest-batch
// and latest-stage first.  Worker threads run the per-frame coder tasks (C1: rANS encode
// y and z, then decode z; C2: decode y).  Batches live in `inflight` slots, each with pinned
// host planes (what the coder reads / writes) and device planes (what the kernels read /
// write).  Three streams: kernels on `stream`, host->device copies on `cstream`,
// device->host copies on `dstream` (symbol planes, and frames when the caller's frames are
// in host memory), ordered by events, so the copies of one batch overlap the kernels of the
// next and the two copy engines run concurrently.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <mutex>
#include <thread>
#include <vector>

#include "../../include/lic.h"
#include "internal.h"

namespace {

using clk = std::chrono::steady_clock;
inline double now_s() { return std::chrono::duration<double>(clk::now().time_since_epoch()).count(); }

enum GpuKind { G_ENC = 0, G_IDX = 1, G_DEC = 2 };
enum CpuKind { C_ONE = 0, C_TWO = 1 };

struct Slot {
    // pinned host planes (coder side)
    int8_t* y_sym = nullptr;  uint8_t* y_idx = nullptr;  int8_t* z_sym = nullptr;
    int8_t* z_dec = nullptr;  uint8_t* idx_dec = nullptr; int8_t* y_dec = nullptr;
    // device planes (kernel side) and frame staging (host frames only)
    int8_t* d_ysym = nullptr; uint8_t* d_yidx = nullptr; int8_t* d_zsym = nullptr;
    int8_t* d_zdec = nullptr; uint8_t* d_idxdec = nullptr; int8_t* d_ydec = nullptr;
    uint8_t* d_fin = nullptr; uint8_t* d_fout = nullptr;
    std::vector<std::vector<uint8_t>> ystr, zstr;
    std::vector<size_t> ylen, zlen;
    // y coded as `parts` slab ranges on separate coder tasks (lic_rans_encode_slab_range)
    std::vector<std::vector<std::vector<uint8_t>>> ypart;   // [frame][part] strings of the part's slabs
    std::vector<std::vector<size_t>> ypart_len;              // [frame][part] bytes
    std::vector<std::vector<uint32_t>> ylens;                // [frame][K] string lengths
    std::vector<int> parts_left;                             // [frame] C_ONE parts still running
    int batch = -1;
    int remaining = 0;
    double t_start = 0;
};

struct GpuTask { GpuKind kind; int slot; double t_ready; };
struct Pending { GpuTask task; cudaEvent_t done; double t_issue; };
constexpr size_t kMaxPendingCap = 16;       // GPU tasks in flight at most (env LIC_MAX_PENDING <= this)
struct CpuTask { CpuKind kind; int slot; int frame; double t_ready; int part = 0; };

}  // namespace

// rans64 tables (cfg.coder = 1): Gaussian rows on the codec's scales (lic_cdf64_gaussian)
struct Tab64 {
    std::vector<uint32_t> cdfs;
    std::vector<int32_t> sizes, offs;
    uint32_t n = 0, stride = 0;
};

static lic_status build_tab64(const lic_codec* codec, int which, Tab64& t) {
    const float* sig = nullptr;
    uint32_t n = 0;
    if (lic_status st = lic_sigmas(codec, which, &sig, &n)) return st;
    float smax = 0.0f;
    for (uint32_t i = 0; i < n; ++i) smax = std::max(smax, sig[i]);
    t.n = n;
    t.stride = 2 * (uint32_t)std::ceil(smax * 6.2f) + 8;     // m(1e-9) = 6.109
    t.cdfs.assign((size_t)n * t.stride, 0u);
    t.sizes.assign(n, 0);
    t.offs.assign(n, 0);
    return lic_cdf64_gaussian(sig, n, 1e-9, t.cdfs.data(), t.stride, t.sizes.data(), t.offs.data());
}

struct lic_pipeline {
    lic_codec* codec = nullptr;
    lic_codec* codec2 = nullptr;            // decoder GPU1 (h_s on decoded z) on its own stream
    cudaStream_t stream2 = nullptr;
    lic_codec* codec3 = nullptr;            // decoder GPU2 (g_s) on its own stream (env LIC_DEC_STREAM=1)
    cudaStream_t stream3 = nullptr;
    lic_pipeline_config cfg{};
    int hyper = 0;
    lic_shape ys{}, zs{};
    size_t ny = 0, nz = 0, in_bytes = 0, out_bytes = 0;
    const uint32_t* cdf_y = nullptr; uint32_t rows_y = 0;
    const uint32_t* cdf_z = nullptr; uint32_t rows_z = 0;
    uint32_t row_len = 0;
    uint32_t ksub = 1;                      // y substreams (channel slabs, lic_rans_encode_slabs)
    uint32_t parts = 1;                     // coder tasks per frame and kind (slab ranges of the y string)
    int sym_min = 0;
    lic_rans_tables* tab_y = nullptr;       // prepared coder tables (lic_rans_prepare)
    lic_rans_tables* tab_z = nullptr;
    uint32_t coder = 0;                     // 0: rANS32 (+ substreams), 1: rans64 + bypass
    Tab64 t64_y, t64_z;
    std::vector<int32_t> ch_rows_y, ch_rows_z;   // channel row of every element (factorized y, z)
    std::vector<Slot> slots;
    std::vector<void*> pinned;
    std::vector<void*> dev;                 // device slot planes
    cudaStream_t stream = nullptr;          // kernels, in issue order
    cudaStream_t cstream = nullptr;         // host -> device copies
    cudaStream_t dstream = nullptr;         // device -> host copies (the other copy engine)
    bool in_host = false, out_host = false; // caller's frames in host memory (staged per slot)
    bool zc = false;                        // codec in zero-copy mode: kernels use the pinned slot planes
    std::vector<cudaEvent_t> events;        // cross-stream join events, recycled as a ring
    std::vector<cudaEvent_t> done_events;   // one per in-flight task (kMaxPendingCap), from a free list
    std::vector<cudaEvent_t> done_free;
    std::deque<Pending> pending;            // issued, not yet completed (FIFO)
    // timeline (cfg.timeline): one record per GPU task / coder task of the last run
    std::vector<lic_timeline_event> tl;
    std::vector<cudaEvent_t> tl_ev;         // timing events: base, then [start, end] per GPU task
    std::vector<std::pair<size_t, size_t>> tl_gpu;   // (record, first event) of every GPU task
    size_t tl_ev_next = 0;
    double t_run0 = 0;
    std::vector<double> slot_free_t;        // when each slot was last released
    // threading
    std::mutex mu;
    std::condition_variable cv_gpu, cv_cpu;
    std::deque<CpuTask> cpu_q;
    std::vector<GpuTask> gpu_q;
    std::vector<std::thread> workers;
    std::condition_variable cv_idle;
    int active = 0;
    bool stop = false;
    // run state
    const uint8_t* in = nullptr;
    uint8_t* out = nullptr;
    int nbatches = 0, next_enc = 0, done = 0;
    std::vector<int> free_slots;
    std::vector<double> lat;
    uint64_t mismatches = 0, y_bytes = 0, z_bytes = 0;
    double coder_busy = 0, gpu_busy = 0;
    lic_status err = LIC_OK;
    std::vector<std::vector<uint8_t>> keep_y, keep_z;
};

// rans64 on int8 planes: symbols / uint8 rows widened to int32 in per-thread buffers
static thread_local std::vector<int32_t> tl_sym, tl_idx;

static const int32_t* rows64(const uint8_t* idx8, const std::vector<int32_t>& ch_rows, size_t n) {
    if (!idx8) return ch_rows.data();
    tl_idx.resize(n);
    for (size_t i = 0; i < n; ++i) tl_idx[i] = idx8[i];
    return tl_idx.data();
}

static lic_status enc64(const Tab64& t, const int8_t* sym, const int32_t* rows, size_t n, std::vector<uint8_t>& out,
                        size_t* len) {
    tl_sym.resize(n);
    for (size_t i = 0; i < n; ++i) tl_sym[i] = sym[i];
    return lic_rans64_encode(tl_sym.data(), rows, n, t.cdfs.data(), t.n, t.stride, t.sizes.data(), t.offs.data(),
                             out.data(), out.size(), len);
}

static lic_status dec64(const Tab64& t, const uint8_t* in, size_t len, const int32_t* rows, size_t n, int8_t* out) {
    tl_sym.resize(n);
    lic_status st = lic_rans64_decode(in, len, rows, n, t.cdfs.data(), t.n, t.stride, t.sizes.data(), t.offs.data(),
                                      tl_sym.data());
    if (st) return st;
    for (size_t i = 0; i < n; ++i) {
        if (tl_sym[i] < -128 || tl_sym[i] > 127) return LIC_ECORRUPT;
        out[i] = (int8_t)tl_sym[i];
    }
    return LIC_OK;
}

static void coder_task64(lic_pipeline* p, const CpuTask& t) {
    Slot& s = p->slots[t.slot];
    const size_t f = (size_t)t.frame;
    lic_status st = LIC_OK;
    uint64_t mism = 0;
    if (t.kind == C_ONE) {
        const int32_t* ry = rows64(p->hyper ? s.y_idx + f * p->ny : nullptr, p->ch_rows_y, p->ny);
        st = enc64(p->t64_y, s.y_sym + f * p->ny, ry, p->ny, s.ystr[f], &s.ylen[f]);
        if (!st && p->hyper)
            st = enc64(p->t64_z, s.z_sym + f * p->nz, p->ch_rows_z.data(), p->nz, s.zstr[f], &s.zlen[f]);
        if (!st && p->hyper) {
            st = dec64(p->t64_z, s.zstr[f].data(), s.zlen[f], p->ch_rows_z.data(), p->nz, s.z_dec + f * p->nz);
            if (!st && std::memcmp(s.z_dec + f * p->nz, s.z_sym + f * p->nz, p->nz) != 0) mism += 1;
        } else if (!st) {
            st = dec64(p->t64_y, s.ystr[f].data(), s.ylen[f], ry, p->ny, s.y_dec + f * p->ny);
            if (!st && std::memcmp(s.y_dec + f * p->ny, s.y_sym + f * p->ny, p->ny) != 0) mism += 1;
        }
    } else {
        const int32_t* ry = rows64(s.idx_dec + f * p->ny, p->ch_rows_y, p->ny);
        st = dec64(p->t64_y, s.ystr[f].data(), s.ylen[f], ry, p->ny, s.y_dec + f * p->ny);
        if (!st && std::memcmp(s.y_dec + f * p->ny, s.y_sym + f * p->ny, p->ny) != 0) mism += 1;
    }
    std::lock_guard<std::mutex> g(p->mu);
    if (st && !p->err) p->err = st;
    p->mismatches += mism;
    if (--s.remaining == 0) {
        if (t.kind == C_ONE && p->hyper) p->gpu_q.push_back({G_IDX, t.slot, now_s()});
        else p->gpu_q.push_back({G_DEC, t.slot, now_s()});
        p->cv_gpu.notify_one();
    }
}

static void coder_task(lic_pipeline* p, const CpuTask& t) {
    if (p->coder == 1) { coder_task64(p, t); return; }
    Slot& s = p->slots[t.slot];
    const size_t f = (size_t)t.frame;
    lic_status st = LIC_OK;
    uint64_t mism = 0;
    bool frame_done = true;                 // this task completes the frame's work of its kind
    if (p->parts > 1) {
        // one slab range [kb, ke) of the y string; part 0 also codes z (encoder) / nothing more
        const uint32_t K = p->ksub, kb = (uint32_t)t.part * K / p->parts, ke = (uint32_t)(t.part + 1) * K / p->parts;
        const size_t hw = (size_t)p->ys.h * p->ys.w;
        const size_t c0 = (size_t)kb * p->ys.c / K, c1 = (size_t)ke * p->ys.c / K;
        if (t.kind == C_ONE) {
            // E(y) of the slabs, and (part 0) E(z) + decoder CPU1 E^-1(z)
            st = lic_rans_encode_slab_range(p->tab_y, s.y_sym + f * p->ny, s.y_idx + f * p->ny, p->ys, K, kb, ke,
                                            s.ypart[f][t.part].data(), s.ypart[f][t.part].size(),
                                            s.ylens[f].data() + kb, &s.ypart_len[f][t.part]);
            if (!st && t.part == 0) {
                st = lic_rans_encode_fast(p->tab_z, s.z_sym + f * p->nz, nullptr, p->zs, s.zstr[f].data(),
                                          s.zstr[f].size(), &s.zlen[f]);
                if (!st) st = lic_rans_decode_fast(p->tab_z, s.zstr[f].data(), s.zlen[f], nullptr, p->zs,
                                                   s.z_dec + f * p->nz);
                if (!st && std::memcmp(s.z_dec + f * p->nz, s.z_sym + f * p->nz, p->nz) != 0) mism += 1;
            }
            bool last = false;
            {
                std::lock_guard<std::mutex> g(p->mu);
                last = --s.parts_left[f] == 0;
            }
            frame_done = last;
            if (last && !st) {
                // the framed string: K big-endian lengths, then the parts in slab order
                uint8_t* w = s.ystr[f].data();
                for (uint32_t k = 0; k < K; ++k) {
                    const uint32_t n = s.ylens[f][k];
                    w[4 * k] = (uint8_t)(n >> 24); w[4 * k + 1] = (uint8_t)(n >> 16);
                    w[4 * k + 2] = (uint8_t)(n >> 8); w[4 * k + 3] = (uint8_t)n;
                }
                size_t pos = 4 * (size_t)K;
                for (uint32_t q = 0; q < p->parts; ++q) {
                    std::memcpy(w + pos, s.ypart[f][q].data(), s.ypart_len[f][q]);
                    pos += s.ypart_len[f][q];
                }
                s.ylen[f] = pos;
            }
        } else {
            // decoder CPU2: E^-1(y) of the slabs with the indexes from decoder GPU1
            st = lic_rans_decode_slab_range(p->tab_y, s.ystr[f].data(), s.ylen[f], s.idx_dec + f * p->ny, p->ys, K,
                                            kb, ke, s.y_dec + f * p->ny);
            if (!st && std::memcmp(s.y_dec + f * p->ny + c0 * hw, s.y_sym + f * p->ny + c0 * hw, (c1 - c0) * hw) != 0)
                mism += 1;
        }
    } else if (t.kind == C_ONE) {
        // encoder CPU workload: E(y) (and E(z)); then decoder CPU1: E^-1(z) (hyper) or E^-1(y)
        st = lic_rans_encode_slabs(p->tab_y, s.y_sym + f * p->ny, p->hyper ? s.y_idx + f * p->ny : nullptr, p->ys,
                                   p->ksub, s.ystr[f].data(), s.ystr[f].size(), &s.ylen[f]);
        if (!st && p->hyper)
            st = lic_rans_encode_fast(p->tab_z, s.z_sym + f * p->nz, nullptr, p->zs, s.zstr[f].data(),
                                      s.zstr[f].size(), &s.zlen[f]);
        if (!st && p->hyper) {
            st = lic_rans_decode_fast(p->tab_z, s.zstr[f].data(), s.zlen[f], nullptr, p->zs, s.z_dec + f * p->nz);
            if (!st && std::memcmp(s.z_dec + f * p->nz, s.z_sym + f * p->nz, p->nz) != 0) mism += 1;
        } else if (!st) {
            st = lic_rans_decode_slabs(p->tab_y, s.ystr[f].data(), s.ylen[f], nullptr, p->ys, p->ksub,
                                       s.y_dec + f * p->ny);
            if (!st && std::memcmp(s.y_dec + f * p->ny, s.y_sym + f * p->ny, p->ny) != 0) mism += 1;
        }
    } else {
        // decoder CPU2: E^-1(y) with the indexes from decoder GPU1
        st = lic_rans_decode_slabs(p->tab_y, s.ystr[f].data(), s.ylen[f], s.idx_dec + f * p->ny, p->ys, p->ksub,
                                   s.y_dec + f * p->ny);
        if (!st && std::memcmp(s.y_dec + f * p->ny, s.y_sym + f * p->ny, p->ny) != 0) mism += 1;
    }
    (void)frame_done;
    std::lock_guard<std::mutex> g(p->mu);
    if (st && !p->err) p->err = st;
    p->mismatches += mism;
    if (--s.remaining == 0) {
        if (t.kind == C_ONE && p->hyper) p->gpu_q.push_back({G_IDX, t.slot, now_s()});
        else p->gpu_q.push_back({G_DEC, t.slot, now_s()});
        p->cv_gpu.notify_one();
    }
}

static void worker_main(lic_pipeline* p, int widx) {
    for (;;) {
        CpuTask t;
        {
            std::unique_lock<std::mutex> lk(p->mu);
            p->cv_cpu.wait(lk, [&] { return p->stop || !p->cpu_q.empty(); });
            if (p->stop) return;
            t = p->cpu_q.front();
            p->cpu_q.pop_front();
            ++p->active;
        }
        const double t0 = now_s();
        const int batch = p->slots[t.slot].batch;
        coder_task(p, t);
        const double t1 = now_s(), dt = t1 - t0;
        std::lock_guard<std::mutex> g(p->mu);
        p->coder_busy += dt;
        if (p->cfg.timeline)
            p->tl.push_back({3u + (uint32_t)t.kind, (uint32_t)widx, batch, t.frame, (t.t_ready - p->t_run0) * 1e3,
                             (t0 - p->t_run0) * 1e3, (t1 - p->t_run0) * 1e3});
        if (--p->active == 0) p->cv_idle.notify_all();
    }
}

extern "C" void lic_pipeline_close(lic_pipeline* p) {
    if (!p) return;
    {
        std::lock_guard<std::mutex> g(p->mu);
        p->stop = true;
    }
    p->cv_cpu.notify_all();
    for (auto& t : p->workers) t.join();
    if (p->stream) cudaStreamSynchronize(p->stream);
    if (p->cstream) cudaStreamSynchronize(p->cstream);
    if (p->dstream) cudaStreamSynchronize(p->dstream);
    if (p->stream2) cudaStreamSynchronize(p->stream2);
    if (p->stream3) cudaStreamSynchronize(p->stream3);
    for (cudaEvent_t e : p->events) cudaEventDestroy(e);
    for (cudaEvent_t e : p->done_events) cudaEventDestroy(e);
    for (cudaEvent_t e : p->tl_ev) cudaEventDestroy(e);
    if (p->stream2) cudaStreamDestroy(p->stream2);
    if (p->codec2) lic_close(p->codec2);
    if (p->stream3) cudaStreamDestroy(p->stream3);
    if (p->codec3) lic_close(p->codec3);
    if (p->stream) cudaStreamDestroy(p->stream);
    if (p->cstream) cudaStreamDestroy(p->cstream);
    if (p->dstream) cudaStreamDestroy(p->dstream);
    for (void* q : p->pinned) cudaFreeHost(q);
    for (void* q : p->dev) cudaFree(q);
    lic_rans_tables_free(p->tab_y);
    lic_rans_tables_free(p->tab_z);
    delete p;
}

extern "C" lic_status lic_pipeline_open(lic_codec* codec, const lic_pipeline_config* cfg, lic_pipeline** out) {
    if (!codec || !cfg || !out || cfg->batch == 0 || cfg->coder_threads == 0) return LIC_EINVAL;
    *out = nullptr;
    lic_pipeline* p = new lic_pipeline();
    p->codec = codec;
    p->cfg = *cfg;
    if (p->cfg.inflight == 0) p->cfg.inflight = 2;
    if (p->cfg.serial) p->cfg.inflight = 1;
    lic_status st = lic_shapes(codec, &p->ys, &p->zs, &p->hyper);
    if (st) { delete p; return st; }
    p->ksub = cfg->substreams ? cfg->substreams : 1;
    // coder tasks per frame: slab ranges of the y string on separate threads (hyperprior,
    // 32-bit rANS with substreams; each range a multiple of 16 slabs keeps the AVX-512 lanes)
    p->parts = cfg->coder_parts ? cfg->coder_parts : 1;
    if (p->parts > 1 && (!p->hyper || cfg->coder != 0 || p->ksub < 2 * p->parts || p->ksub % p->parts)) p->parts = 1;
    p->zc = lic_internal_zero_copy(codec) != 0;
    if (p->ksub > 64 || p->ksub > p->ys.c) { delete p; return LIC_EINVAL; }
    p->ny = (size_t)p->ys.c * p->ys.h * p->ys.w;
    p->nz = (size_t)p->zs.c * p->zs.h * p->zs.w;
    uint32_t rl = 0;
    if (p->hyper) {
        if ((st = lic_cdf(codec, 2, &p->cdf_y, &p->rows_y, &rl)) || (st = lic_cdf(codec, 1, &p->cdf_z, &p->rows_z, &rl))) {
            delete p;
            return st;
        }
    } else if ((st = lic_cdf(codec, 0, &p->cdf_y, &p->rows_y, &rl))) {
        delete p;
        return st;
    }
    p->row_len = rl;
    p->sym_min = -(int)((rl - 2) / 2);
    if ((st = lic_rans_prepare(p->cdf_y, p->rows_y, rl, p->sym_min, &p->tab_y)) ||
        (p->hyper && (st = lic_rans_prepare(p->cdf_z, p->rows_z, rl, p->sym_min, &p->tab_z)))) {
        lic_pipeline_close(p);
        return st;
    }
    p->coder = cfg->coder;
    if (p->coder > 1) { lic_pipeline_close(p); return LIC_EINVAL; }
    if (p->coder == 1) {
        if ((st = build_tab64(codec, p->hyper ? 2 : 0, p->t64_y)) ||
            (p->hyper && (st = build_tab64(codec, 1, p->t64_z)))) {
            lic_pipeline_close(p);
            return st;
        }
        auto ch_rows = [](const lic_shape& sh, std::vector<int32_t>& r) {
            r.resize((size_t)sh.c * sh.h * sh.w);
            for (size_t i = 0; i < r.size(); ++i) r[i] = (int32_t)(i / ((size_t)sh.h * sh.w));
        };
        if (!p->hyper) ch_rows(p->ys, p->ch_rows_y);
        else ch_rows(p->zs, p->ch_rows_z);
    }
    const size_t B = cfg->batch;
    auto pin = [&](size_t bytes) -> void* {
        void* q = nullptr;
        if (cudaHostAlloc(&q, bytes ? bytes : 16, cudaHostAllocMapped | cudaHostAllocPortable) != cudaSuccess) {
            cudaGetLastError();
            return nullptr;
        }
        p->pinned.push_back(q);
        return q;
    };
    auto dalloc = [&](size_t bytes) -> void* {
        void* q = nullptr;
        if (cudaMalloc(&q, bytes ? bytes : 16) != cudaSuccess) {
            cudaGetLastError();
            return nullptr;
        }
        p->dev.push_back(q);
        return q;
    };
    const size_t fbytes = B * lic_internal_frame_pixels(codec) * 3 * (cfg->u8 ? 1 : 4);
    p->slots.resize(p->cfg.inflight);
    for (Slot& s : p->slots) {
        s.d_ysym = (int8_t*)dalloc(B * p->ny);
        s.d_ydec = (int8_t*)dalloc(B * p->ny);
        s.d_yidx = (uint8_t*)dalloc(p->hyper ? B * p->ny : 16);
        s.d_idxdec = (uint8_t*)dalloc(p->hyper ? B * p->ny : 16);
        s.d_zsym = (int8_t*)dalloc(p->hyper ? B * p->nz : 16);
        s.d_zdec = (int8_t*)dalloc(p->hyper ? B * p->nz : 16);
        s.d_fin = (uint8_t*)dalloc(fbytes);
        s.d_fout = (uint8_t*)dalloc(fbytes);
        if (!s.d_ysym || !s.d_ydec || !s.d_yidx || !s.d_idxdec || !s.d_zsym || !s.d_zdec || !s.d_fin || !s.d_fout) {
            lic_pipeline_close(p);
            return LIC_ENOMEM;
        }
        s.y_sym = (int8_t*)pin(B * p->ny);
        s.y_dec = (int8_t*)pin(B * p->ny);
        s.y_idx = (uint8_t*)pin(p->hyper ? B * p->ny : 16);
        s.idx_dec = (uint8_t*)pin(p->hyper ? B * p->ny : 16);
        s.z_sym = (int8_t*)pin(p->hyper ? B * p->nz : 16);
        s.z_dec = (int8_t*)pin(p->hyper ? B * p->nz : 16);
        if (!s.y_sym || !s.y_dec || !s.y_idx || !s.idx_dec || !s.z_sym || !s.z_dec) {
            lic_pipeline_close(p);
            return LIC_ENOMEM;
        }
        // rans64: <= 16 bits per symbol plus <= 12 escape bits (int8 values), words of 4 bytes
        const size_t ycap = p->coder == 1 ? 4 * p->ny + 64 : 2 * p->ny + 64 + 8 * p->ksub;
        const size_t zcap = p->coder == 1 ? 4 * p->nz + 64 : 2 * p->nz + 64;
        s.ystr.assign(B, std::vector<uint8_t>(ycap));
        s.ypart.assign(B, std::vector<std::vector<uint8_t>>(p->parts, std::vector<uint8_t>(ycap)));
        s.ypart_len.assign(B, std::vector<size_t>(p->parts, 0));
        s.ylens.assign(B, std::vector<uint32_t>(p->ksub, 0));
        s.parts_left.assign(B, 0);
        s.zstr.assign(B, std::vector<uint8_t>(zcap));
        s.ylen.assign(B, 0);
        s.zlen.assign(B, 0);
    }
    if (cudaStreamCreateWithFlags(&p->stream, cudaStreamNonBlocking) != cudaSuccess ||
        cudaStreamCreateWithFlags(&p->cstream, cudaStreamNonBlocking) != cudaSuccess ||
        cudaStreamCreateWithFlags(&p->dstream, cudaStreamNonBlocking) != cudaSuccess) {
        cudaGetLastError();
        lic_pipeline_close(p);
        return LIC_ECUDA;
    }
    // decoder GPU1 (three small h_s launches per batch) on a second codec and stream, so its
    // kernels can fill the SMs other batches' kernels leave idle (env LIC_IDX_STREAM=0: off)
    {
        const char* e = std::getenv("LIC_IDX_STREAM");
        if (p->hyper && !p->cfg.serial && !(e && e[0] == '0')) {
            if ((st = lic_internal_clone(codec, &p->codec2)) != LIC_OK ||
                cudaStreamCreateWithFlags(&p->stream2, cudaStreamNonBlocking) != cudaSuccess) {
                cudaGetLastError();
                lic_pipeline_close(p);
                return st ? st : LIC_ECUDA;
            }
        }
    }
    // decoder GPU2 on a third codec and stream: its kernels may share the GPU with the next
    // batches' encode kernels (env LIC_DEC_STREAM=1: on)
    {
        const char* e = std::getenv("LIC_DEC_STREAM");
        if (!p->cfg.serial && e && e[0] == '1') {
            if ((st = lic_internal_clone(codec, &p->codec3)) != LIC_OK ||
                cudaStreamCreateWithFlags(&p->stream3, cudaStreamNonBlocking) != cudaSuccess) {
                cudaGetLastError();
                lic_pipeline_close(p);
                return st ? st : LIC_ECUDA;
            }
        }
    }
    // join events only order streams (a wait captures the event when it is enqueued, so the
    // ring may recycle them); a task's completion event is waited on later by the control
    // thread and must not be re-recorded before then: those come from their own free list
    p->events.resize(32);
    p->done_events.resize(kMaxPendingCap);
    for (auto* v : {&p->events, &p->done_events})
        for (auto& e : *v)
            if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) {
                cudaGetLastError();
                lic_pipeline_close(p);
                return LIC_ECUDA;
            }
    p->done_free = p->done_events;
    for (uint32_t i = 0; i < cfg->coder_threads; ++i) p->workers.emplace_back(worker_main, p, (int)i);
    *out = p;
    return LIC_OK;
}

// cstream -> stream -> cstream ordering through recycled events (a wait captures the event's
// state when it is enqueued, so re-recording an event later is harmless)
static cudaEvent_t next_event(lic_pipeline* p, size_t& ev_next) { return p->events[ev_next++ % p->events.size()]; }
static bool join(lic_pipeline* p, cudaStream_t from, cudaStream_t to, size_t& ev_next) {
    cudaEvent_t e = next_event(p, ev_next);
    return cudaEventRecord(e, from) == cudaSuccess && cudaStreamWaitEvent(to, e, 0) == cudaSuccess;
}

// Issues one GPU task: H2D inputs (cstream), kernels (stream), D2H outputs (cstream); returns
// with `done` recorded after the last step.
static lic_status gpu_call(lic_pipeline* p, const GpuTask& t, cudaEvent_t done, size_t& ev_next) {
    Slot& s = p->slots[t.slot];
    const uint32_t B = p->cfg.batch;
    const size_t b = (size_t)s.batch;
    const size_t fb = (size_t)B * p->in_bytes;
    lic_status st = LIC_OK;
    auto cp = [&](void* dst, const void* src, size_t n, cudaMemcpyKind k) {
        cudaStream_t cs = k == cudaMemcpyHostToDevice ? p->cstream : p->dstream;
        if (!st && cudaMemcpyAsync(dst, src, n, k, cs) != cudaSuccess) st = LIC_ECUDA;
    };
    auto to_k = [&]() { if (!st && !join(p, p->cstream, p->stream, ev_next)) st = LIC_ECUDA; };
    // timeline: device timestamps around the task's kernels on the stream they run on
    const bool tl = p->cfg.timeline && p->tl_ev_next + 2 <= p->tl_ev.size();
    size_t ev0 = 0;
    auto mark = [&](cudaStream_t ks, int end) {
        if (!tl || st) return;
        if (!end) ev0 = p->tl_ev_next;
        if (cudaEventRecord(p->tl_ev[p->tl_ev_next++], ks) != cudaSuccess) st = LIC_ECUDA;
    };
    auto to_c = [&]() { if (!st && !join(p, p->stream, p->dstream, ev_next)) st = LIC_ECUDA; };
    switch (t.kind) {
    case G_ENC: {
        const uint8_t* fr = p->in + b * fb;
        if (p->in_host) { cp(s.d_fin, fr, fb, cudaMemcpyHostToDevice); to_k(); fr = s.d_fin; }
        // zero-copy: the epilogues write the pinned slot planes in place
        int8_t* ys = p->zc ? s.y_sym : s.d_ysym;
        uint8_t* yi = p->zc ? s.y_idx : s.d_yidx;
        int8_t* zs = p->zc ? s.z_sym : s.d_zsym;
        mark(p->stream, 0);
        if (!st)
            st = p->cfg.u8 ? lic_encode_u8(p->codec, fr, B, ys, p->hyper ? yi : nullptr, p->hyper ? zs : nullptr,
                                           nullptr, p->stream)
                           : lic_encode(p->codec, (const float*)fr, B, ys, p->hyper ? yi : nullptr,
                                        p->hyper ? zs : nullptr, nullptr, p->stream);
        mark(p->stream, 1);
        to_c();
        if (!p->zc) {
            cp(s.y_sym, s.d_ysym, B * p->ny, cudaMemcpyDeviceToHost);
            if (p->hyper) {
                cp(s.y_idx, s.d_yidx, B * p->ny, cudaMemcpyDeviceToHost);
                cp(s.z_sym, s.d_zsym, B * p->nz, cudaMemcpyDeviceToHost);
            }
        }
        break;
    }
    case G_IDX: {
        lic_codec* cc = p->codec2 ? p->codec2 : p->codec;
        cudaStream_t ks = p->codec2 ? p->stream2 : p->stream;
        if (!p->zc) cp(s.d_zdec, s.z_dec, B * p->nz, cudaMemcpyHostToDevice);
        if (!st && !join(p, p->cstream, ks, ev_next)) st = LIC_ECUDA;
        mark(ks, 0);
        if (!st)
            st = lic_hyper_indexes(cc, p->zc ? s.z_dec : s.d_zdec, B, p->zc ? s.idx_dec : s.d_idxdec, ks);
        mark(ks, 1);
        if (!st && !join(p, ks, p->dstream, ev_next)) st = LIC_ECUDA;
        if (!p->zc) cp(s.idx_dec, s.d_idxdec, B * p->ny, cudaMemcpyDeviceToHost);
        break;
    }
    case G_DEC: {
        lic_codec* cc = p->codec3 ? p->codec3 : p->codec;
        cudaStream_t ks = p->codec3 ? p->stream3 : p->stream;
        if (!p->zc) cp(s.d_ydec, s.y_dec, B * p->ny, cudaMemcpyHostToDevice);
        if (!st && !join(p, p->cstream, ks, ev_next)) st = LIC_ECUDA;
        uint8_t* fr = p->out + b * fb;
        uint8_t* dst = p->out_host ? s.d_fout : fr;
        const int8_t* yd = p->zc ? s.y_dec : s.d_ydec;
        mark(ks, 0);
        if (!st)
            st = p->cfg.u8 ? lic_decode_u8(cc, yd, B, dst, ks)
                           : lic_decode(cc, yd, B, (float*)dst, ks);
        mark(ks, 1);
        if (!st && !join(p, ks, p->dstream, ev_next)) st = LIC_ECUDA;
        if (p->out_host) cp(fr, s.d_fout, fb, cudaMemcpyDeviceToHost);
        break;
    }
    }
    // every task ends with kernels -> dstream (possibly no copies after them)
    if (!st && cudaEventRecord(done, p->dstream) != cudaSuccess) st = LIC_ECUDA;
    if (tl && !st) {
        std::lock_guard<std::mutex> g(p->mu);
        p->tl_gpu.push_back({p->tl.size(), ev0});
        p->tl.push_back({(uint32_t)t.kind, (uint32_t)(t.kind == G_IDX && p->codec2 ? 1 : (t.kind == G_DEC && p->codec3 ? 2 : 0)), s.batch, -1,
                         (t.t_ready - p->t_run0) * 1e3, 0.0, 0.0});
    }
    return st;
}

static bool is_host(const void* q) {
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, q) != cudaSuccess) { cudaGetLastError(); return true; }
    return a.type != cudaMemoryTypeDevice && a.type != cudaMemoryTypeManaged;
}

extern "C" lic_status lic_pipeline_run(lic_pipeline* p, const void* frames_in, uint32_t nframes, void* frames_out,
                                       lic_pipeline_stats* stats) {
    if (!p || !frames_in || !frames_out || nframes == 0 || nframes % p->cfg.batch) return LIC_EINVAL;
    const uint32_t B = p->cfg.batch;
    const size_t px = lic_internal_frame_pixels(p->codec);
    p->in_bytes = px * 3 * (p->cfg.u8 ? 1 : 4);
    p->out_bytes = p->in_bytes;
    {
        std::lock_guard<std::mutex> g(p->mu);
        p->in = (const uint8_t*)frames_in;
        p->out = (uint8_t*)frames_out;
        p->in_host = is_host(frames_in);
        p->out_host = is_host(frames_out);
        p->nbatches = (int)(nframes / B);
        p->next_enc = 0;
        p->done = 0;
        p->free_slots.clear();
        for (int i = (int)p->slots.size() - 1; i >= 0; --i) p->free_slots.push_back(i);
        p->gpu_q.clear();
        p->cpu_q.clear();
        p->pending.clear();
        p->lat.clear();
        p->mismatches = p->y_bytes = p->z_bytes = 0;
        p->coder_busy = p->gpu_busy = 0;
        p->err = LIC_OK;
        if (p->cfg.keep_bitstreams) {
            p->keep_y.assign(nframes, {});
            p->keep_z.assign(nframes, {});
        }
    }
    const uint64_t launches0 = lic_internal_launches(p->codec) + lic_internal_launches(p->codec2) +
                               lic_internal_launches(p->codec3);
    // timeline: a base event, then two timing events per GPU task
    p->tl.clear();
    p->tl_gpu.clear();
    p->tl_ev_next = 0;
    if (p->cfg.timeline) {
        const size_t need = 1 + 2 * (size_t)p->nbatches * (p->hyper ? 3 : 2);
        while (p->tl_ev.size() < need) {
            cudaEvent_t e;
            if (cudaEventCreate(&e) != cudaSuccess) { cudaGetLastError(); return LIC_ECUDA; }
            p->tl_ev.push_back(e);
        }
    }
    p->slot_free_t.assign(p->slots.size(), 0.0);
    const double t_run0 = now_s();
    p->t_run0 = t_run0;
    if (p->cfg.timeline) {
        if (cudaEventRecord(p->tl_ev[0], p->stream) != cudaSuccess) return LIC_ECUDA;
        p->tl_ev_next = 1;
    }
    // paced submission (cfg.pace_fps > 0): batch i is submitted at t_run0 + i * batch / pace_fps
    // and its latency counts from then (queueing included); unpaced, every frame is there
    // at the start and latency counts from the batch's admission into a slot
    const double pace = p->cfg.pace_fps > 0 ? (double)p->cfg.pace_fps : 0.0;
    auto t_submit = [&](int i) { return t_run0 + (double)i * (double)B / pace; };
    // GPU control loop.  GPU tasks are issued asynchronously on p->stream (at most
    // kMaxPending in flight, env LIC_MAX_PENDING) so the device never idles while ready work exists; the
    // oldest issued task is retired by waiting on its event, which then releases its
    // coder tasks (ENC, IDX) or its slot (DEC).
    size_t kMaxPending = 5;
    if (const char* e = std::getenv("LIC_MAX_PENDING"))
        kMaxPending = (size_t)std::max(1, std::min((int)kMaxPendingCap, atoi(e)));
    p->done_free = p->done_events;
    size_t ev_next = 0;
    for (;;) {
        GpuTask t{};
        bool issue = false;
        {
            std::unique_lock<std::mutex> lk(p->mu);
            auto can_enc = [&] {
                if (p->next_enc >= p->nbatches || p->free_slots.empty()) return false;
                if (pace > 0 && now_s() < t_submit(p->next_enc)) return false;
                return !p->cfg.serial || p->done == p->next_enc;
            };
            auto have_ready = [&] { return !p->gpu_q.empty() || can_enc(); };
            auto wake = [&] { return p->err || p->done == p->nbatches || !p->pending.empty() || have_ready(); };
            if (pace > 0 && p->next_enc < p->nbatches) {
                // sleep at most until the next submission is due
                const auto due = clk::time_point(std::chrono::duration_cast<clk::duration>(
                    std::chrono::duration<double>(t_submit(p->next_enc))));
                p->cv_gpu.wait_until(lk, due, wake);
                if (!wake()) continue;
            } else {
                p->cv_gpu.wait(lk, wake);
            }
            if (p->err || p->done == p->nbatches) break;
            if (p->pending.size() < kMaxPending && have_ready()) {
                issue = true;
                if (!p->gpu_q.empty()) {
                    // latest stage first, then oldest batch: drains frames, bounds latency
                    auto best = std::max_element(p->gpu_q.begin(), p->gpu_q.end(),
                                                 [&](const GpuTask& a, const GpuTask& b) {
                                                     if (a.kind != b.kind) return a.kind < b.kind;
                                                     return p->slots[a.slot].batch > p->slots[b.slot].batch;
                                                 });
                    t = *best;
                    p->gpu_q.erase(best);
                } else {
                    const int s = p->free_slots.back();
                    p->free_slots.pop_back();
                    const int bi = p->next_enc++;
                    p->slots[s].batch = bi;
                    p->slots[s].t_start = pace > 0 ? t_submit(bi) : now_s();
                    t = {G_ENC, s, std::max(pace > 0 ? t_submit(bi) : t_run0, p->slot_free_t[s])};
                }
            }
        }
        if (issue) {
            const double g0 = now_s();
            cudaEvent_t ev = p->done_free.back();          // pending.size() < kMaxPending <= cap
            p->done_free.pop_back();
            lic_status st = gpu_call(p, t, ev, ev_next);
            std::lock_guard<std::mutex> g(p->mu);
            if (st) { p->err = st; break; }
            p->pending.push_back({t, ev, g0});
            continue;
        }
        // nothing issuable: retire the oldest in-flight GPU task
        Pending pd;
        {
            std::lock_guard<std::mutex> g(p->mu);
            pd = p->pending.front();
            p->pending.pop_front();
        }
        const double w0 = now_s();
        const cudaError_t ce = cudaEventSynchronize(pd.done);
        const double g1 = now_s();
        std::lock_guard<std::mutex> g(p->mu);
        p->done_free.push_back(pd.done);
        p->gpu_busy += g1 - std::max(w0, pd.t_issue);
        if (ce != cudaSuccess) { p->err = LIC_ECUDA; break; }
        t = pd.task;
        Slot& s = p->slots[t.slot];
        if (t.kind == G_ENC || t.kind == G_IDX) {
            s.remaining = (int)(B * p->parts);
            for (uint32_t f = 0; f < B; ++f) {
                if (t.kind == G_ENC) s.parts_left[f] = (int)p->parts;
                for (uint32_t q = 0; q < p->parts; ++q)
                    p->cpu_q.push_back({t.kind == G_ENC ? C_ONE : C_TWO, t.slot, (int)f, g1, (int)q});
            }
            p->cv_cpu.notify_all();
        } else {
            for (uint32_t f = 0; f < B; ++f) {
                p->y_bytes += s.ylen[f];
                p->z_bytes += p->hyper ? s.zlen[f] : 0;
                if (p->cfg.keep_bitstreams) {
                    const size_t gi = (size_t)s.batch * B + f;
                    p->keep_y[gi].assign(s.ystr[f].begin(), s.ystr[f].begin() + s.ylen[f]);
                    if (p->hyper) p->keep_z[gi].assign(s.zstr[f].begin(), s.zstr[f].begin() + s.zlen[f]);
                }
            }
            p->lat.push_back((g1 - s.t_start) * 1e3);
            p->slot_free_t[t.slot] = g1;
            p->free_slots.push_back(t.slot);
            ++p->done;
        }
    }
    // leave nothing running on the streams
    cudaStreamSynchronize(p->stream);
    if (p->stream2) cudaStreamSynchronize(p->stream2);
    if (p->stream3) cudaStreamSynchronize(p->stream3);
    cudaStreamSynchronize(p->cstream);
    cudaStreamSynchronize(p->dstream);
    const double t_run1 = now_s();
    if (p->cfg.timeline && !p->err) {
        for (const auto& g : p->tl_gpu) {
            float a = 0, b = 0;
            cudaEventElapsedTime(&a, p->tl_ev[0], p->tl_ev[g.second]);
            cudaEventElapsedTime(&b, p->tl_ev[0], p->tl_ev[g.second + 1]);
            p->tl[g.first].t_start_ms = a;
            p->tl[g.first].t_end_ms = b;
        }
    }
    // error path: drop queued coder work and wait for tasks already running
    std::unique_lock<std::mutex> g(p->mu);
    p->cpu_q.clear();
    p->cv_idle.wait(g, [&] { return p->active == 0; });
    if (stats) {
        std::memset(stats, 0, sizeof *stats);
        stats->frames = (uint64_t)p->done * B;
        stats->seconds = t_run1 - t_run0;
        std::vector<double> l = p->lat;
        std::sort(l.begin(), l.end());
        if (!l.empty()) {
            stats->latency_p50_ms = l[l.size() / 2];
            stats->latency_p95_ms = l[std::min(l.size() - 1, (size_t)(0.95 * l.size()))];
            stats->latency_max_ms = l.back();
        }
        stats->y_bytes = p->y_bytes;
        stats->z_bytes = p->z_bytes;
        stats->symbol_mismatches = p->mismatches;
        stats->gpu_busy_s = p->gpu_busy;
        stats->coder_busy_s = p->coder_busy;
        stats->gpu_launches = lic_internal_launches(p->codec) + lic_internal_launches(p->codec2) +
                              lic_internal_launches(p->codec3) - launches0;
    }
    return p->err;
}

extern "C" lic_status lic_pipeline_timeline(const lic_pipeline* p, lic_timeline_event* out, size_t cap, size_t* n) {
    if (!p || !n) return LIC_EINVAL;
    if (!p->cfg.timeline) return LIC_EINVAL;
    *n = p->tl.size();
    if (out) std::memcpy(out, p->tl.data(), std::min(cap, p->tl.size()) * sizeof(lic_timeline_event));
    return cap < p->tl.size() && out ? LIC_ENOSPACE : LIC_OK;
}

extern "C" lic_status lic_pipeline_bitstream(const lic_pipeline* p, uint32_t frame, const uint8_t** y, size_t* y_len,
                                             const uint8_t** z, size_t* z_len) {
    if (!p || !p->cfg.keep_bitstreams || frame >= p->keep_y.size()) return LIC_EINVAL;
    if (y) *y = p->keep_y[frame].data();
    if (y_len) *y_len = p->keep_y[frame].size();
    if (z) *z = p->hyper ? p->keep_z[frame].data() : nullptr;
    if (z_len) *z_len = p->hyper ? p->keep_z[frame].size() : 0;
    return LIC_OK;
}
