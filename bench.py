#!/usr/bin/env python
"""bench.py -- throughput of the learned-image-codec hot path on B200.

Metric (BASELINE.json): "1280x720 encode+decode frames/s at 1/2/4/8 B200; p50 frame
latency; % TC peak".  Workload: configs[2] of BASELINE.json -- scale-hyperprior N=128
M=192, 1280x720 synthetic video stream (padded to 1280x768), random-init weights
(lic_synth), synthetic u8 frames.

A step = one batch of B frames through the whole hot path:
GPU encode (g_a, h_a, Q(z), h_s, sigma->index) -> host rANS encode of y and z -> host
rANS decode of z (decoder CPU1) -> GPU hyper_indexes (decoder GPU1) -> host rANS decode of
y (decoder CPU2) -> GPU decode (g_s) -- through the native pipeline (lic_pipeline_run):
one GPU control thread plus a pool of coder threads, batches in flight so GPU work and the
host coder overlap (§III).

  value : frames/s, input frames resident in HBM, decoded frames written to HBM; the timed
          run has no profiling events at all.
  e2e   : frames/s with frames read from / written to pinned host memory through the same
          C-ABI call (host<->device copies inside the timed region).
Sub-measurements: every layer against its own roofline (tensor or HBM),
the dominant kernel timed in a separate pass, transform-only GPU fps, host-coder Msym/s per
thread, the overlap criterion e2e >= 0.9 min(GPU-only, coder-only), the GPU idle time
while work was ready (pipeline timeline), paced submit -> complete latency, the serial
reference, a full-frame oracle timing, and the C4 configuration.
Multi-GPU (torchrun): frame t of the stream belongs to rank t mod G (weak scaling, no
collective on the data path); time = max over ranks.

--impl reference: the CPU oracle (oracle/) on the host cores, a bounded sample per step.
"""
from __future__ import annotations

import argparse
import json
import os
import platform
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CODERS = {"rans32": 0, "rans64": 1}
CONFIGS = {
    "c2": dict(kind=0, N=128, M=192, H=512, W=768, B=1,
               workload="factorized-prior N=128 M=192, Kodak-shaped 768x512 frames, batch 1, random-init weights"),
    "c3": dict(kind=1, N=128, M=192, H=720, W=1280, B=4,
               workload="scale-hyperprior N=128 M=192, 1280x720 synthetic stream (padded 1280x768), random-init weights"),
    "c4": dict(kind=1, N=192, M=320, H=720, W=1280, B=4,
               workload="scale-hyperprior N=192 M=320, 1280x720 synthetic stream (padded 1280x768), random-init weights"),
    "c5": dict(kind=1, N=192, M=320, H=1080, W=1920, B=2,
               workload="scale-hyperprior N=192 M=320, 1920x1080 synthetic stream (padded 1920x1088), random-init weights"),
}
STREAM_SEED, STREAM_T = 1000, 8     # frame t of the stream = synth_frame_u8(seed 1000, t mod 8), any rank
HBM_LAYERS = ("ga1", "gs4")        # K = 75 / N = 3: below the ridge point


def padded(h, w, hyper):
    P = 64 if hyper else 16
    return -(-h // P) * P, -(-w // P) * P


# ----------------------------------------------------------------- algorithmic work
def layer_flops(cfg):
    """Algorithmic FLOPs (2 x MAC) per frame of every GEMM-engine layer, including the
    GDN/IGDN gamma contraction (C^2 MACs per pixel).  conv: Ho*Wo*Cout*Cin*k^2; deconv:
    Hi*Wi*Cin*Cout*k^2."""
    N, M = cfg["N"], cfg["M"]
    Hp, Wp = padded(cfg["H"], cfg["W"], cfg["kind"] == 1)
    H2, W2 = Hp // 2, Wp // 2
    f = {}

    def conv(name, ho, wo, cin, cout, k, gdn=False):
        f[name] = 2 * ho * wo * cout * cin * k * k + (2 * ho * wo * cout * cout if gdn else 0)
    conv("ga1", H2, W2, 3, N, 5, True)
    conv("ga2", H2 // 2, W2 // 2, N, N, 5, True)
    conv("ga3", H2 // 4, W2 // 4, N, N, 5, True)
    conv("ga4", Hp // 16, Wp // 16, N, M, 5)
    conv("ha1", Hp // 16, Wp // 16, M, N, 3)
    conv("ha2", Hp // 32, Wp // 32, N, N, 5)
    conv("ha3", Hp // 64, Wp // 64, N, N, 5)

    def deconv(name, hi, wi, cin, cout, gdn=False):     # deconv MACs counted on the input grid
        f[name] = 2 * hi * wi * cin * cout * 25 + (2 * 4 * hi * wi * cout * cout if gdn else 0)
    deconv("hs1", Hp // 64, Wp // 64, N, N)
    deconv("hs2", Hp // 32, Wp // 32, N, N)
    conv("hs3", Hp // 16, Wp // 16, N, M, 3)
    deconv("gs1", Hp // 16, Wp // 16, M, N, True)
    deconv("gs2", Hp // 8, Wp // 8, N, N, True)
    deconv("gs3", Hp // 4, Wp // 4, N, N, True)
    deconv("gs4", H2, W2, N, 3)
    return f


def layer_bytes(cfg, split=2):
    """Algorithmic HBM bytes per frame of the HBM-bound layers: one read of the input and one
    write of the output.  g_a L1: the u8 frame in, the fp16 hi + lo activation out; g_s L4:
    the hi + lo activation in, the u8 frame out."""
    Hp, Wp = padded(cfg["H"], cfg["W"], cfg["kind"] == 1)
    act = (Hp // 2) * (Wp // 2) * cfg["N"] * 2 * split
    frame = cfg["H"] * cfg["W"] * 3
    return {"ga1": frame + act, "gs4": act + frame}


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return json.load(fh), "measured"
    except OSError:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


def layer_roofline(cfg, name, ms_per_launch, batch, pk, split=2):
    """(bound, achieved, peak, unit, frac) of one launch of layer `name`."""
    if name in HBM_LAYERS:
        gbs = layer_bytes(cfg, split)[name] * batch / (ms_per_launch / 1e3) / 1e9
        return "hbm", gbs, pk["hbm_gbs"], "GB/s", gbs / pk["hbm_gbs"]
    tf = layer_flops(cfg)[name] * batch / (ms_per_launch / 1e3) / 1e12
    peak = pk.get("bf16_tflops_sustained", 1400.0)
    return "tensor", tf, peak, "TFLOP/s", tf / peak


# ----------------------------------------------------------------- clocks
class ClockSampler:
    """SM clocks and clock-event (throttle) reasons sampled in-process through NVML every
    2 ms while the timed region runs (a 40 ms region still gets ~20 samples)."""
    REASONS = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20,
               "sw_power_cap": 0x4, "hw_power_brake": 0x80}

    def __init__(self, local):
        self.local = local
        self.samples = []
        self.reasons = 0
        self.max_mhz = None
        self._stop = threading.Event()
        self.h = None

    def __enter__(self):
        try:
            import pynvml as N
            import torch
            N.nvmlInit()
            self.N = N
            try:
                pr = torch.cuda.get_device_properties(self.local)
                bus = f"{pr.pci_domain_id:08x}:{pr.pci_bus_id:02x}:{pr.pci_device_id:02x}.0"
                self.h = N.nvmlDeviceGetHandleByPciBusId(bus)
            except Exception:
                self.h = N.nvmlDeviceGetHandleByIndex(self.local)
            self.max_mhz = N.nvmlDeviceGetMaxClockInfo(self.h, N.NVML_CLOCK_SM)
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        except Exception:
            self.h = None
        return self

    def _run(self):
        N = self.N
        while not self._stop.is_set():
            try:
                self.samples.append(N.nvmlDeviceGetClockInfo(self.h, N.NVML_CLOCK_SM))
                self.reasons |= N.nvmlDeviceGetCurrentClocksEventReasons(self.h)
            except Exception:
                pass
            time.sleep(0.002)

    def __exit__(self, *a):
        self._stop.set()
        if self.h is not None:
            self.t.join(timeout=2)

    def summary(self):
        return {"sm_mhz": float(np.median(self.samples)) if self.samples else None,
                "sm_max_mhz": self.max_mhz,
                "reasons": sorted(k for k, v in self.REASONS.items() if self.reasons & v),
                "samples": len(self.samples), "source": "NVML in-process, 2 ms period"}


# ----------------------------------------------------------------- oracle (CPU baseline)
def cpu_model():
    try:
        with open("/proc/cpuinfo") as fh:
            for ln in fh:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor() or "unknown"


def oracle_full_frame(cfg):
    """The oracle as it stands on one whole frame of the workload (frame 0 of the stream):
    encode (transforms, quantiser, sigma -> index), rANS encode, rANS decode, decode."""
    from lic_synth import ModelSpec, generate_weights, synth_frame_u8
    from oracle import oracle as O
    hyper = cfg["kind"] == 1
    spec = ModelSpec(kind=cfg["kind"], N=cfg["N"], M=cfg["M"])
    w = generate_weights(spec, seed=0)
    t = O.build_tables(w, hyper, 32)
    fr = synth_frame_u8(cfg["H"], cfg["W"], seed=STREAM_SEED, t=0)
    t0 = time.perf_counter()
    x, crop = O.ingest_u8(fr, hyper=hyper)
    p = O.encode_planes(x, w, hyper, 32)
    t1 = time.perf_counter()
    yb, zb = O.code_planes(p, t, hyper)
    O.decode_strings(yb, zb, w, t, hyper, p["y_sym"].shape, p["z_sym"].shape if hyper else None, crop,
                     cfg["H"], cfg["W"])
    dt = time.perf_counter() - t0
    cores = int(os.environ.get("OMP_NUM_THREADS", len(os.sched_getaffinity(0))))
    return 1.0 / dt, cores, (f"one whole {cfg['W']}x{cfg['H']} frame: oracle encode + rANS encode/decode + decode, "
                             f"{dt:.1f} s ({t1 - t0:.1f} s encode), {cores} OpenMP threads on {cpu_model()}")


# ----------------------------------------------------------------- per-rank cores
def bind_rank_cores(local, world):
    """One process per GPU shares the host: give local rank r its own contiguous slice of the
    cores it may run on, so each rank's coder pool and GPU control thread stay off the others'
    cores (env LIC_BIND_CORES=0: no binding).  Returns the slice (or None)."""
    if world <= 1 or os.environ.get("LIC_BIND_CORES", "1") == "0" or not hasattr(os, "sched_setaffinity"):
        return None
    cores = sorted(os.sched_getaffinity(0))
    per = len(cores) // world
    if per < 2:
        return None
    mine = cores[local * per:(local + 1) * per]
    os.sched_setaffinity(0, mine)
    return mine


# ----------------------------------------------------------------- timeline analysis
def idle_while_ready(tl, t_end_ms):
    """Time the GPU executed nothing while some GPU task was ready (its inputs done, not yet
    started): the overlap evidence of SURVEY.md §8(d).  Returns (ms, busy ms)."""
    gpu = [e for e in tl if e["kind"].startswith("gpu")]
    edges = []
    for e in gpu:
        edges.append((e["start"], 0, +1))                 # busy
        edges.append((e["end"], 0, -1))
        if e["start"] > e["ready"]:
            edges.append((e["ready"], 1, +1))             # waiting
            edges.append((e["start"], 1, -1))
    edges.sort(key=lambda x: x[0])
    busy = wait = 0
    idle_ready = busy_ms = 0.0
    prev = 0.0
    for t, kind, d in edges:
        t = min(max(t, 0.0), t_end_ms)
        if busy == 0 and wait > 0:
            idle_ready += t - prev
        if busy > 0:
            busy_ms += t - prev
        prev = t
        if kind == 0:
            busy += d
        else:
            wait += d
    return idle_ready, busy_ms


def chrome_trace(tl, path):
    ev = []
    for e in tl:
        gpu = e["kind"].startswith("gpu")
        ev.append({"name": f"{e['kind']} b{e['batch']}" + ("" if gpu else f" f{e['frame']}"), "ph": "X",
                   "pid": "GPU" if gpu else "coder", "tid": e["lane"], "ts": e["start"] * 1e3,
                   "dur": max(0.0, e["end"] - e["start"]) * 1e3})
    with open(path, "w") as fh:
        json.dump({"traceEvents": ev, "displayTimeUnit": "ms"}, fh)


# ----------------------------------------------------------------- one configuration
def measure(args, name, rank, world, local, threads, full):
    import torch
    import torch.distributed as dist
    from lic_synth import ModelSpec, generate_weights, synth_frames_u8, write_licw
    from paper_2208_01641_b200 import lic

    cfg = CONFIGS[name]
    H, W = cfg["H"], cfg["W"]
    B = args.batch if (args.batch and name == args.config) else cfg["B"]
    # default run: >= 3000 frames; the driver passes --steps explicitly
    steps = (args.steps or -(-3000 // B)) if full else max(10, min(args.steps or 40, 40))
    split = 2 if args.precision == "split" else 1
    spec = ModelSpec(kind=cfg["kind"], N=cfg["N"], M=cfg["M"], activation=1 if args.activation == "1dn" else 0)
    blob = write_licw(spec, generate_weights(spec, seed=0))
    codec = lic.Codec(blob, H, W, max_batch=B, device=local,
                      precision=lic.PREC_F16 if args.precision == "f16" else lic.PREC_SPLIT)
    codec.set_zero_copy(args.zero_copy)
    mk = dict(coder_threads=threads, batch=B, u8=True, substreams=args.substreams, coder=CODERS[args.coder],
              coder_parts=args.coder_parts)
    pipe = lic.Pipeline(codec, inflight=args.inflight, **mk)

    # the stream: local frame i of rank r is global frame t = r + G*i (frame t mod 8 of seed 1000)
    base = torch.from_numpy(synth_frames_u8(STREAM_T, H, W, seed=STREAM_SEED))
    nfr = steps * B
    # frames held on the device (and pinned on the host): at most ~2.8 GB of u8 frames; longer
    # runs push the same buffer through again (one lic_pipeline_run call per pass, run_n)
    nbuf = min(nfr, max(B, (int(2.8e9) // (H * W * 3)) // B * B))
    nloc = max(nbuf, args.warmup * B)
    gidx = (rank + world * torch.arange(nloc)) % STREAM_T
    dev_in = base[gidx].cuda()                                  # frames resident in HBM
    dev_out = torch.empty_like(dev_in)
    host_in = base[gidx].pin_memory()
    host_out = torch.empty_like(host_in).pin_memory()
    frame_bytes = H * W * 3

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()

    def run_n(p, src, dst, n):
        """n frames through the pipeline, in passes over the nbuf frames on the device."""
        agg, done = None, 0
        while done < n:
            k = min(nbuf, n - done)
            s_ = p.run(src, dst, k)
            if agg is None:
                agg = dict(s_)
            else:
                for key in ("frames", "seconds", "y_bytes", "z_bytes", "symbol_mismatches", "gpu_busy_s",
                            "coder_busy_s", "gpu_launches"):
                    agg[key] += s_[key]
                for key in ("latency_p95_ms", "latency_max_ms"):
                    agg[key] = max(agg[key], s_[key])
            done += k
        return agg

    def timed(p, src, dst, n, clocks=None):
        barrier()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        if clocks:
            clocks.__enter__()
        ev0.record()
        st = run_n(p, src, dst, n)
        ev1.record()
        torch.cuda.synchronize()
        if clocks:
            clocks.__exit__()
        ms = ev0.elapsed_time(ev1)
        barrier()
        return ms, st

    def max_over_ranks(v):
        if world == 1:
            return v
        t = torch.tensor([v], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    pipe.run(dev_in, dev_out, args.warmup * B)                  # warm-up (untimed)

    # ---- 1. untimed pass, every GEMM-engine launch bracketed by events: per-layer times and
    # roofline fractions (events between kernels serialise them: a conservative split)
    nprof = min(nfr, 64 * B)
    codec.profile(True)
    ms_prof, _ = timed(pipe, dev_in, dev_out, nprof)
    prof_all = codec.profile_read()
    codec.profile(False)
    dom = max(prof_all, key=lambda k: prof_all[k][0])

    # ---- 2. the timed run (value): no profiling events
    clocks = ClockSampler(local)
    ms, st = timed(pipe, dev_in, dev_out, nfr, clocks)
    if st["symbol_mismatches"]:
        raise SystemExit(f"lossless round trip failed: {st['symbol_mismatches']} frames")
    launches = st["gpu_launches"]

    # ---- 3. the dominant kernel alone bracketed by events (its own pass)
    codec.profile(True, layers=[dom])
    ms_dom_run, _ = timed(pipe, dev_in, dev_out, nfr)
    prof = codec.profile_read()
    codec.profile(False)

    # ---- 4. end to end through pinned host buffers
    ms_e2e, st_e2e = timed(pipe, host_in, host_out, nfr)

    ms = max_over_ranks(ms)
    ms_e2e = max_over_ranks(ms_e2e)
    total = nfr * world
    value = total / (ms / 1e3)
    e2e = total / (ms_e2e / 1e3)

    pk, pk_src = peaks()
    dom_ms, dom_n = prof[dom]
    per_launch_ms = dom_ms / dom_n
    bound, ach, peak, unit, frac = layer_roofline(cfg, dom, per_launch_ms, B, pk, split)
    traffic = None
    try:        # DRAM bytes per launch from the committed ncu --set full capture (the C3 workload)
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as fh:
            traffic = json.load(fh).get(dom) if name == "c3" else None
    except (OSError, ValueError, AttributeError):
        pass
    layers = {}
    for k, (lms, ln) in sorted(prof_all.items(), key=lambda kv: -kv[1][0]):
        b_, a_, p_, u_, f_ = layer_roofline(cfg, k, lms / ln, B, pk, split)
        layers[k] = {"share": round(lms / ms_prof, 4), "ms_per_launch": round(lms / ln, 4), "bound": b_,
                     "achieved": round(a_, 1), "unit": u_, "frac": round(f_, 4)}

    ny = int(np.prod(codec.y_shape))
    nz = int(np.prod(codec.z_shape)) if codec.hyper else 0
    # PCIe bytes per step in the e2e run: frames in/out (DMA) + symbol planes through pinned
    # slots: encode writes y_sym, y_idx, z_sym; GPU1 reads z_dec, writes idx_dec; GPU2 reads y_dec
    h2d = B * (frame_bytes + nz + ny)
    d2h = B * (frame_bytes + 2 * ny + nz + ny)

    res = {
        "value": value, "e2e": e2e, "ms": ms, "steps": steps, "B": B, "nfr": nfr, "launches": launches,
        "workload": cfg["workload"], "st": st, "clocks": clocks.summary(), "h2d": h2d, "d2h": d2h,
        "roofline": {"bound": bound, "kernel": f"conv_umma_kernel[{dom}]", "achieved": round(ach, 2),
                     "peak": peak, "unit": unit, "frac": round(frac, 4), "traffic": traffic,
                     "peak_source": (f"{pk_src} " + ("hbm_gbs" if bound == "hbm" else
                                                      "bf16_tflops_sustained (fp16 dense rate = bf16)")),
                     "algorithmic_per_launch": (layer_bytes(cfg, split)[dom] if bound == "hbm" else
                                                layer_flops(cfg)[dom]) * B,
                     "avg_launch_ms": round(per_launch_ms, 4),
                     "timing": f"CUDA events around the {dom} launches only, in a run of its own",
                     "note": ("split-FP16 issues 2 MMAs per algorithmic FLOP: tensor ceiling frac 0.5"
                              if split == 2 else "single fp16 plane: 1 MMA per algorithmic FLOP")},
        "layers": layers,
    }
    if not full:
        pipe.close()
        codec.close()
        return res

    # ---- 5. transform-only GPU fps: encode -> hyper_indexes -> decode, no coder
    s = torch.cuda.Stream()
    ys = torch.empty((B,) + codec.y_shape, dtype=torch.int8, device="cuda")
    yi = torch.empty((B,) + codec.y_shape, dtype=torch.uint8, device="cuda") if codec.hyper else None
    zs = torch.empty((B,) + codec.z_shape, dtype=torch.int8, device="cuda") if codec.hyper else None
    yi2 = torch.empty_like(yi) if codec.hyper else None
    fo = torch.empty((B, H, W, 3), dtype=torch.uint8, device="cuda")

    def gpu_step(i):
        fr = dev_in[(i * B) % nbuf:(i * B) % nbuf + B]
        codec.encode(fr, ys, yi, zs, stream=s, u8=True)
        if codec.hyper:
            codec.hyper_indexes(zs, yi2, stream=s)
        codec.decode(ys, fo, stream=s, u8=True)
    with torch.cuda.stream(s):
        for i in range(3):
            gpu_step(i)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for i in range(steps):
            gpu_step(i)
        e1.record(s)
        torch.cuda.synchronize()
    gpu_only = steps * B / (e0.elapsed_time(e1) / 1e3)

    # ---- 6. host coder, one thread: Msym/s and ms per frame (E(y), E(z), E^-1(z), E^-1(y))
    yh, zh = ys.cpu().numpy(), (zs.cpu().numpy() if codec.hyper else None)
    ih = yi.cpu().numpy() if codec.hyper else None
    ty = lic.RansTables(codec.cdf(2 if codec.hyper else 0))
    tz = lic.RansTables(codec.cdf(1)) if codec.hyper else None
    K = args.substreams
    reps = max(3, 20 // B)
    t0 = time.perf_counter()
    for _ in range(reps):
        for f in range(B):
            yb = ty.encode(yh[f], ih[f] if codec.hyper else None, substreams=K)
            if codec.hyper:
                zb = tz.encode(zh[f])
                tz.decode(zb, zh[f].shape)
            ty.decode(yb, yh[f].shape, ih[f] if codec.hyper else None, substreams=K)
    coder_s = (time.perf_counter() - t0) / (reps * B)
    msym = 2 * (ny + nz) / coder_s / 1e6
    coder_only = threads / coder_s
    try:
        import ctypes
        avx = "avx512f" in open("/proc/cpuinfo").read() and os.environ.get("LIC_NO_AVX512") != "1"
    except OSError:
        avx = False

    # ---- 7. pipeline timeline (untimed): GPU idle while work was ready
    tp = lic.Pipeline(codec, inflight=args.inflight, timeline=True, **mk)
    ntl = min(nbuf, 48 * B)
    t_tl0 = time.perf_counter()
    tp.run(dev_in, dev_out, ntl)
    tl_ms = (time.perf_counter() - t_tl0) * 1e3
    tl = tp.timeline()
    tp.close()
    idle_ms, busy_ms = idle_while_ready(tl, tl_ms)
    if args.timeline_out:
        chrome_trace(tl, args.timeline_out)

    # ---- 8. paced source: submit -> complete latency at 80 % of the measured per-GPU rate
    pace = 0.8 * value / world
    pp = lic.Pipeline(codec, inflight=args.inflight, pace_fps=pace, **mk)
    npace = min(nloc, max(B * 4, int(pace * 1.0) // B * B))     # ~1 s of frames, within the device set
    stp = pp.run(dev_in, dev_out, npace)
    pp.close()

    # ---- 9. serial reference (no overlap between stages)
    sp = lic.Pipeline(codec, inflight=1, serial=True, **mk)
    nser = min(nbuf, 16 * B)
    t0 = time.perf_counter()
    sp.run(dev_in, dev_out, nser)
    serial_fps = nser / (time.perf_counter() - t0)
    sp.close()

    res.update({
        "gpu_only_fps": gpu_only, "coder_s_per_frame": coder_s, "coder_msym_s": msym, "coder_only_fps": coder_only,
        "avx512": avx, "idle_ready_ms": idle_ms, "busy_ms": busy_ms, "tl_ms": tl_ms, "tl_frames": ntl,
        "pace": pace, "paced": stp, "npace": npace, "serial_fps": serial_fps, "e2e_st": st_e2e,
    })

    # ---- 10. end-of-run bitstream gather (off the timed loop): global frames 0..7, whoever
    # holds them, ordered by index on rank 0 -- the digest is the same for every G
    from paper_2208_01641_b200.dist import gather_bitstreams, stream_digest, verify_frames
    nv, keep = verify_frames(rank, world, B, STREAM_T)
    vp = lic.Pipeline(codec, inflight=2, keep_bitstreams=True, **mk)
    vst = vp.run(dev_in, dev_out, nv)
    local_bs = {t: vp.bitstream(i) for i, t in keep}
    vp.close()
    merged = gather_bitstreams(local_bs, rank, world)
    res["bitstreams"] = None if merged is None else {
        "frames_gathered": len(merged), "global_frames": f"0..{STREAM_T - 1}", "sha256": stream_digest(merged),
        "lossless": vst["symbol_mismatches"] == 0}
    pipe.close()
    codec.close()
    return res


# ----------------------------------------------------------------- main
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=0,
                    help="timed steps (batches); 0: >= 3000 frames (reference arm: 5 bounded samples)")
    ap.add_argument("--warmup", type=int, default=8, help="untimed warm-up steps (8 x 4 frames >= SPEC.md:452's 30)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c3", choices=sorted(CONFIGS),
                    help="BASELINE.json config (c3: the headline 720p hyperprior stream)")
    ap.add_argument("--also", default="c4", help="comma-separated extra configs measured briefly ('' = none)")
    ap.add_argument("--batch", type=int, default=0, help="frames per step (per GPU); 0: the config's")
    ap.add_argument("--coder-threads", type=int, default=0, help="0: derived from the host cores")
    ap.add_argument("--inflight", type=int, default=8)
    ap.add_argument("--substreams", type=int, default=32,
                    help="y string as K channel-slab rANS substreams (DESIGN.md R21); 1 = one string")
    ap.add_argument("--coder-parts", type=int, default=2,
                    help="coder tasks per frame: the y string's slab ranges on separate threads (same bitstream)")
    ap.add_argument("--coder", default="rans32", choices=["rans32", "rans64"],
                    help="host entropy coder: 32-bit rANS over +-L tables (with --substreams), or rans64 + "
                         "bypass escape with Gaussian tables (DESIGN.md R23; one string per plane)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--zero-copy", action="store_true", help="kernels touch pinned host planes in place")
    ap.add_argument("--activation", default="gdn", choices=["gdn", "1dn"],
                    help="g_a / g_s normalisation: GDN, or the paper's 1DN (implementation C, PAPER.md:131-137)")
    ap.add_argument("--precision", default="split", choices=["split", "f16"],
                    help="split: fp16 hi + lo activations (graded); f16: one fp16 plane (NEXT-4, ungraded)")
    ap.add_argument("--timeline-out", default="", help="write the pipeline timeline as a Chrome trace JSON")
    args = ap.parse_args()
    assert args.warmup >= 3 or args.impl == "reference", "timing rules: >= 3 warm-up steps"

    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))

    if args.impl == "reference":
        return run_reference(args, rank, world)

    import torch
    import torch.distributed as dist
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    ncores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 8)
    bound = bind_rank_cores(local, world)
    cores = len(bound) if bound else max(1, ncores // max(1, world))
    threads = args.coder_threads or max(2, min(96, cores - 2))

    r = measure(args, args.config, rank, world, local, threads, full=True)
    cfg = CONFIGS[args.config]
    st = r["st"]
    line = {
        "metric": f"{cfg['W']}x{cfg['H']} encode+decode frames/s",
        "value": round(r["value"], 2),
        "unit": "frames/s",
        "n_gpus": world,
        "steps": r["steps"],
        "warmup": args.warmup,
        "ms_per_step": round(r["ms"] / r["steps"], 3),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f16x2(split hi/lo)->f32" if args.precision == "split" else "f16->f32 (single plane, ungraded)",
        "data": "synthetic",
        "config": {"workload": r["workload"] + (", 1DN activation" if args.activation == "1dn" else ""),
                   "batch_per_gpu": r["B"], "frames_per_gpu": r["nfr"], "world": world,
                   "coder_threads_per_gpu": threads, "cores_per_rank": cores, "inflight": args.inflight,
                   "y_substreams": args.substreams if args.coder == "rans32" else 1, "entropy_coder": args.coder,
                   "coder_parts": args.coder_parts,
                   "l2": "inputs larger than L2 (activations ~0.36 GB per frame, frame set > 126 MB)",
                   "pipeline": "overlapped"},
        "latency_ms": {"p50": round(r["paced"]["latency_p50_ms"], 3), "p95": round(r["paced"]["latency_p95_ms"], 3),
                       "max": round(r["paced"]["latency_max_ms"], 3),
                       "definition": (f"per batch, submission -> decoded frames in HBM, queueing included, paced "
                                      f"source at {r['pace']:.0f} frames/s per GPU (80 % of value), "
                                      f"{r['npace']} frames"),
                       "unpaced_service_p50": round(st["latency_p50_ms"], 3)},
        "bits": {"y_bytes_per_frame": st["y_bytes"] / r["nfr"], "z_bytes_per_frame": st["z_bytes"] / r["nfr"],
                 "bpp": 8 * (st["y_bytes"] + st["z_bytes"]) / r["nfr"] / (cfg["H"] * cfg["W"])},
        "roofline": r["roofline"],
        "layers": r["layers"],
        "layers_note": "untimed pass with every layer bracketed by events; tensor layers vs the sustained "
                       "fp16 dense peak, g_a L1 / g_s L4 vs HBM",
        "gpu_launches": int(r["launches"]),
        "e2e": {"value": round(r["e2e"], 2), "unit": "frames/s", "h2d_bytes_per_step": r["h2d"],
                "d2h_bytes_per_step": r["d2h"]},
        "overlap": {
            "gpu_only_fps": round(r["gpu_only_fps"], 1),
            "coder_ms_per_frame_1thread": round(r["coder_s_per_frame"] * 1e3, 3),
            "coder_msym_s_per_thread": round(r["coder_msym_s"], 1),
            "coder_threads": threads, "coder_avx512": r["avx512"],
            "coder_only_fps": round(r["coder_only_fps"], 1),
            "criterion": "e2e >= 0.9 * min(gpu_only, coder_only)",
            "criterion_met": bool(r["e2e"] / world >= 0.9 * min(r["gpu_only_fps"], r["coder_only_fps"])),
            "gpu_idle_while_ready_ms": round(r["idle_ready_ms"], 3),
            "gpu_busy_ms": round(r["busy_ms"], 3),
            "timeline_ms": round(r["tl_ms"], 3),
            "timeline_note": f"lic_pipeline_timeline of an untimed {r['tl_frames']}-frame run (device times of "
                             "every GPU task, host times of every coder task)",
            "serial_reference_fps": round(r["serial_fps"], 1),
        },
        "clocks": r["clocks"],
    }
    for extra in [x for x in args.also.split(",") if x and x != args.config]:
        e = measure(args, extra, rank, world, local, threads, full=False)
        line.setdefault("other_configs", {})[extra] = {
            "workload": e["workload"], "value": round(e["value"], 2), "e2e": round(e["e2e"], 2),
            "steps": e["steps"], "batch_per_gpu": e["B"], "roofline": e["roofline"], "clocks": e["clocks"]}
    if rank == 0:
        line["bitstreams"] = r["bitstreams"]
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        v, c, desc = oracle_full_frame(cfg)
        line["cpu_baseline"] = {"value": round(v, 6), "unit": "frames/s", "cores": c, "kind": "oracle",
                                "sample": desc}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def run_reference(args, rank, world):
    """Reference arm: the CPU oracle, as it stands, on this box's host cores."""
    if rank != 0:
        return
    cfg = CONFIGS[args.config]
    H, W = cfg["H"], cfg["W"]
    steps, warm = args.steps or 5, args.warmup
    # each step: a bounded sample (one 1280x64 strip = 1/12 of a padded 720p frame)
    from lic_synth import ModelSpec, generate_weights, synth_frame_u8
    from oracle import oracle as O
    hyper = cfg["kind"] == 1
    spec = ModelSpec(kind=cfg["kind"], N=cfg["N"], M=cfg["M"])
    w = generate_weights(spec, seed=0)
    t = O.build_tables(w, hyper, 32)
    rows = 64

    def step(i):
        fr = synth_frame_u8(rows, W, seed=2000 + i)
        x, crop = O.ingest_u8(fr, hyper=hyper)
        p = O.encode_planes(x, w, hyper, 32)
        yb, zb = O.code_planes(p, t, hyper)
        O.decode_strings(yb, zb, w, t, hyper, p["y_sym"].shape, p["z_sym"].shape if hyper else None, crop, rows, W)

    for i in range(min(warm, 1)):
        step(i)
    t0 = time.perf_counter()
    for i in range(steps):
        step(i)
    dt = time.perf_counter() - t0
    frames = steps * rows / float(padded(H, W, hyper)[0])
    v = frames / dt
    cores = int(os.environ.get("OMP_NUM_THREADS", len(os.sched_getaffinity(0))))
    desc = (f"{steps} steps x oracle encode+decode of a {W}x{rows} strip ({rows}/{padded(H, W, hyper)[0]} of a "
            f"padded frame), {cores} threads on {cpu_model()}")
    line = {"impl": "reference", "metric": f"{W}x{H} encode+decode frames/s", "value": round(v, 6),
            "unit": "frames/s", "n_gpus": world, "steps": steps, "warmup": warm, "ms_per_step": round(dt / steps * 1e3, 3),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64 accumulate / f32",
            "data": "synthetic", "config": {"workload": cfg["workload"] + " (oracle, bounded strip sample per step)"},
            "cpu_baseline": {"value": round(v, 6), "unit": "frames/s", "cores": cores, "kind": "oracle", "sample": desc},
            "e2e": {"value": round(v, 6), "unit": "frames/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
