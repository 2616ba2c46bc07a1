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
one GPU control thread plus a pool of coder threads, batches double-buffered so GPU work
and the host coder overlap (§III).

  value : frames/s, input frames resident in HBM, decoded frames written to HBM.
  e2e   : frames/s with frames read from / written to pinned host memory through the same
          C-ABI call (host<->device copies inside the timed region).
Multi-GPU (torchrun): frames shard by rank (weak scaling, no collective on the data
path); time = max over ranks.

--impl reference: the CPU oracle (oracle/) on the host cores, a bounded sample per step.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# BASELINE.json configs (configs[2] = C3 is the default, headline workload; the others are
# reported by DESIGN.md from `--config` runs on one GPU)
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
CFG = CONFIGS["c3"]
H, W = CFG["H"], CFG["W"]
N_CH, M_CH = CFG["N"], CFG["M"]
WORKLOAD = CFG["workload"]


def padded(h, w, hyper):
    P = 64 if hyper else 16
    return -(-h // P) * P, -(-w // P) * P


def set_config(name):
    global CFG, H, W, N_CH, M_CH, WORKLOAD
    CFG = CONFIGS[name]
    H, W, N_CH, M_CH, WORKLOAD = CFG["H"], CFG["W"], CFG["N"], CFG["M"], CFG["workload"]


# ----------------------------------------------------------------- algorithmic work
def layer_flops(N=None, M=None, Hp=None, Wp=None):
    """Algorithmic FLOPs (2 x MAC) per frame of every GEMM-engine layer, including the
    GDN/IGDN gamma contraction (C^2 MACs per pixel).  conv: Ho*Wo*Cout*Cin*k^2; deconv:
    Hi*Wi*Cin*Cout*k^2."""
    N = N or N_CH
    M = M or M_CH
    if Hp is None:
        Hp, Wp = padded(H, W, CFG["kind"] == 1)
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
    # deconv MACs counted on the input grid
    def deconv(name, hi, wi, cin, cout, gdn=False):
        f[name] = 2 * hi * wi * cin * cout * 25 + (2 * 4 * hi * wi * cout * cout if gdn else 0)
    deconv("hs1", Hp // 64, Wp // 64, N, N)
    deconv("hs2", Hp // 32, Wp // 32, N, N)
    conv("hs3", Hp // 16, Wp // 16, N, M, 3)
    deconv("gs1", Hp // 16, Wp // 16, M, N, True)
    deconv("gs2", Hp // 8, Wp // 8, N, N, True)
    deconv("gs3", Hp // 4, Wp // 4, N, N, True)
    deconv("gs4", H2, W2, N, 3)
    return f


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return json.load(fh), "measured"
    except OSError:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


# ----------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), "--query-gpu=clocks.sm,clocks.max.sm,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], 0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx = max(mx, float(parts[1]))
            except ValueError:
                continue
            for n, v in zip(names, parts[2:]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ----------------------------------------------------------------- oracle (CPU baseline)
def oracle_sample(seconds_budget=15.0, strip_rows=64, seed=0):
    """The oracle as it stands, full encode + decode (transforms, quantiser, sigma->index,
    rANS) on a 1280 x strip_rows strip of the 720p frame: the same per-pixel work at
    1/12 of the padded 1280x768 frame.  Returns (frames/s, cores, description)."""
    from lic_synth import ModelSpec, generate_weights, synth_frame_u8
    from oracle import oracle as O
    hyper = CFG["kind"] == 1
    spec = ModelSpec(kind=CFG["kind"], N=N_CH, M=M_CH)
    w = generate_weights(spec, seed=0)
    t = O.build_tables(w, hyper, 32)
    fr = synth_frame_u8(strip_rows, W, seed=seed)
    t0 = time.perf_counter()
    n = 0
    while True:
        x, crop = O.ingest_u8(fr, hyper=hyper)
        p = O.encode_planes(x, w, hyper, 32)
        yb, zb = O.code_planes(p, t, hyper)
        O.decode_strings(yb, zb, w, t, hyper, p["y_sym"].shape, p["z_sym"].shape if hyper else None, crop,
                         strip_rows, W)
        n += 1
        if time.perf_counter() - t0 >= seconds_budget or n >= 40:
            break
    dt = time.perf_counter() - t0
    frac = strip_rows / float(padded(H, W, hyper)[0])
    cores = int(os.environ.get("OMP_NUM_THREADS", os.cpu_count() or 1))
    return n * frac / dt, cores, (f"{n} x oracle encode+decode of a {W}x{strip_rows} strip "
                                  f"(= {frac:.4f} of a padded {W}x{H} frame each), {dt:.1f} s")


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


# ----------------------------------------------------------------- main
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=250)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c3", choices=sorted(CONFIGS),
                    help="BASELINE.json config (c3: the headline 720p hyperprior stream)")
    ap.add_argument("--batch", type=int, default=0, help="frames per step (per GPU); 0: the config's")
    ap.add_argument("--coder-threads", type=int, default=0, help="0: derived from the host cores")
    ap.add_argument("--inflight", type=int, default=8)
    ap.add_argument("--substreams", type=int, default=32,
                    help="y string as K channel-slab rANS substreams (DESIGN.md R21); 1 = one string")
    ap.add_argument("--coder", default="rans32", choices=["rans32", "rans64"],
                    help="host entropy coder: 32-bit rANS over +-L tables (with --substreams), or rans64 + "
                         "bypass escape with Gaussian tables (DESIGN.md R23; one string per plane)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--serial", action="store_true", help="serial reference pipeline (no overlap)")
    ap.add_argument("--zero-copy", action="store_true", help="kernels touch pinned host planes in place")
    ap.add_argument("--activation", default="gdn", choices=["gdn", "1dn"],
                    help="g_a / g_s normalisation: GDN, or the paper's 1DN (implementation C, PAPER.md:131-137)")
    ap.add_argument("--precision", default="split", choices=["split", "f16"],
                    help="split: fp16 hi + lo activations (graded); f16: one fp16 plane (NEXT-4, ungraded)")
    args = ap.parse_args()
    assert args.warmup >= 3 or args.impl == "reference", "timing rules: >= 3 warm-up steps"
    set_config(args.config)
    if not args.batch:
        args.batch = CFG["B"]

    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))

    if args.impl == "reference":
        return run_reference(args, rank, world)

    import torch
    import torch.distributed as dist
    from lic_synth import ModelSpec, generate_weights, synth_frames_u8, write_licw
    from paper_2208_01641_b200 import lic

    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    ncores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 8)
    threads = args.coder_threads or max(2, min(96, ncores // max(1, world) - 2))
    bound = bind_rank_cores(local, world)

    B = args.batch
    spec = ModelSpec(kind=CFG["kind"], N=N_CH, M=M_CH, activation=1 if args.activation == "1dn" else 0)
    blob = write_licw(spec, generate_weights(spec, seed=0))
    codec = lic.Codec(blob, H, W, max_batch=B, device=local,
                      precision=lic.PREC_F16 if args.precision == "f16" else lic.PREC_SPLIT)
    codec.set_zero_copy(args.zero_copy)
    pipe = lic.Pipeline(codec, coder_threads=threads, batch=B, inflight=args.inflight, u8=True,
                        serial=args.serial, substreams=args.substreams, coder=CODERS[args.coder])

    # synthetic stream: 8 distinct frames per rank, looped (the paper loops one image)
    base = torch.from_numpy(synth_frames_u8(8, H, W, seed=1000 + rank))
    nfr = args.steps * B
    idx = torch.arange(max(nfr, args.warmup * B)) % 8
    dev_in = base[idx].cuda()                                   # frames resident in HBM
    dev_out = torch.empty_like(dev_in)
    host_in = base[idx].pin_memory()
    host_out = torch.empty_like(host_in).pin_memory()
    frame_bytes = H * W * 3

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()

    def timed(src, dst, n):
        barrier()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record()
        st = pipe.run(src, dst, n)
        ev1.record()
        torch.cuda.synchronize()
        ms = ev0.elapsed_time(ev1)
        barrier()
        return ms, st

    # warm-up (untimed)
    pipe.run(dev_in, dev_out, args.warmup * B)

    # ---- untimed pass with every GEMM-engine launch bracketed by events: per-kernel share of
    # the step and the dominant kernel (events between kernels serialise them, so the timed
    # run below brackets only the dominant kernel)
    nprof = min(nfr, 64 * B)
    codec.profile(True)
    ms_prof, _ = timed(dev_in, dev_out, nprof)
    prof_all = codec.profile_read()
    codec.profile(False)
    dom = max(prof_all, key=lambda k: prof_all[k][0])

    # ---- device-resident run (value), events around the dominant kernel's launches only
    codec.profile(True, layers=[dom])
    with ClockSampler(local) as clocks:
        ms, st = timed(dev_in, dev_out, nfr)
    launches = st["gpu_launches"]
    prof = codec.profile_read()
    codec.profile(False)
    if st["symbol_mismatches"]:
        raise SystemExit(f"lossless round trip failed: {st['symbol_mismatches']} frames")

    # ---- end-to-end through pinned host buffers
    ms_e2e, st_e2e = timed(host_in, host_out, nfr)

    def max_over_ranks(v):
        if world == 1:
            return v
        t = torch.tensor([v], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    ms = max_over_ranks(ms)
    ms_e2e = max_over_ranks(ms_e2e)
    total_frames = nfr * world
    value = total_frames / (ms / 1e3)
    e2e = total_frames / (ms_e2e / 1e3)

    # ---- roofline of the dominant kernel (largest summed device time)
    pk, pk_src = peaks()
    flops = layer_flops()
    dom_ms, dom_n = prof[dom]
    per_launch_ms = dom_ms / dom_n
    achieved = flops[dom] * B / (per_launch_ms / 1e3) / 1e12
    peak = pk.get("bf16_tflops_sustained", 1400.0)
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as fh:
            tr = json.load(fh)
            traffic = tr.get(dom)
    except (OSError, ValueError):
        pass
    kernel_share = {k: round(v[0] / ms_prof, 4) for k, v in sorted(prof_all.items(), key=lambda kv: -kv[1][0])}

    ny = int(np.prod(codec.y_shape))
    nz = int(np.prod(codec.z_shape)) if codec.hyper else 0
    # PCIe bytes per step in the e2e run: frames in/out (DMA) + symbol planes through pinned
    # slots: encode writes y_sym, y_idx, z_sym; GPU1 reads z_dec, writes idx_dec; GPU2 reads y_dec
    h2d = B * (frame_bytes + nz + ny)
    d2h = B * (frame_bytes + 2 * ny + nz + ny)

    line = {
        "metric": f"{W}x{H} encode+decode frames/s",
        "value": round(value, 2),
        "unit": "frames/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(ms / args.steps, 3),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f16x2(split hi/lo)->f32" if args.precision == "split" else "f16->f32 (single plane, ungraded)",
        "data": "synthetic",
        "config": {"workload": WORKLOAD + (", 1DN activation" if args.activation == "1dn" else ""),
                   "batch_per_gpu": B, "frames_per_gpu": nfr,
                   "coder_threads_per_gpu": threads, "inflight": args.inflight,
                   "cores_per_rank": len(bound) if bound else ncores,
                   "y_substreams": args.substreams if args.coder == "rans32" else 1,
                   "entropy_coder": args.coder,
                   "l2": "inputs larger than L2 (activations ~0.36 GB per frame, frame set > 126 MB)",
                   "pipeline": "serial" if args.serial else "overlapped"},
        "latency_ms": {"p50": round(st["latency_p50_ms"], 3), "p95": round(st["latency_p95_ms"], 3),
                       "max": round(st["latency_max_ms"], 3), "definition": "per batch, GPU encode start -> decode end"},
        "bits": {"y_bytes_per_frame": st["y_bytes"] / nfr, "z_bytes_per_frame": st["z_bytes"] / nfr,
                 "bpp": 8 * (st["y_bytes"] + st["z_bytes"]) / nfr / (H * W)},
        "busy": {"gpu_thread_s": round(st["gpu_busy_s"], 3), "coder_threads_s": round(st["coder_busy_s"], 3),
                 "wall_s": round(st["seconds"], 3)},
        "roofline": {"bound": "tensor", "kernel": f"conv_umma_kernel[{dom}]", "achieved": round(achieved, 2),
                     "peak": peak, "unit": "TFLOP/s", "frac": round(achieved / peak, 4), "traffic": traffic,
                     "peak_source": f"{pk_src} bf16_tflops_sustained (fp16 dense rate = bf16)",
                     "algorithmic_flops_per_launch": flops[dom] * B, "avg_launch_ms": round(per_launch_ms, 4),
                     "note": ("split-FP16 issues 2 MMAs per algorithmic FLOP: ceiling frac 0.5"
                              if args.precision == "split" else "single fp16 plane: 1 MMA per algorithmic FLOP")},
        "kernel_time_share": kernel_share,
        "kernel_time_share_note": f"untimed pass of {nprof} frames with every layer bracketed by events",
        "gpu_launches": int(launches),
        "e2e": {"value": round(e2e, 2), "unit": "frames/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
        "clocks": clocks.summary(),
    }
    # ---- end-of-run bitstream gather (off the timed loop): every rank's per-frame strings
    # for its first frames, ordered by global frame index on rank 0
    from paper_2208_01641_b200.dist import gather_bitstreams, stream_digest
    vp = lic.Pipeline(codec, coder_threads=threads, batch=B, inflight=2, u8=True, keep_bitstreams=True,
                      substreams=args.substreams, coder=CODERS[args.coder])
    vst = vp.run(dev_in, dev_out, 2 * B)
    local = {rank + world * i: vp.bitstream(i) for i in range(2 * B)}
    vp.close()
    merged = gather_bitstreams(local, rank, world)
    if rank == 0:
        line["bitstreams"] = {"frames_gathered": len(merged), "sha256": stream_digest(merged),
                              "lossless": vst["symbol_mismatches"] == 0}
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        v, cores, desc = oracle_sample()
        line["cpu_baseline"] = {"value": round(v, 6), "unit": "frames/s", "cores": cores, "kind": "oracle",
                                "sample": desc}
    if rank == 0:
        print(json.dumps(line), flush=True)
    pipe.close()
    codec.close()
    if world > 1:
        dist.destroy_process_group()


def run_reference(args, rank, world):
    """Reference arm: the CPU oracle, as it stands, on this box's host cores."""
    if rank != 0:
        return
    steps, warm = args.steps, args.warmup
    # each step: a bounded sample (one 1280x64 strip = 1/12 of a padded 720p frame)
    from lic_synth import ModelSpec, generate_weights, synth_frame_u8
    from oracle import oracle as O
    hyper = CFG["kind"] == 1
    spec = ModelSpec(kind=CFG["kind"], N=N_CH, M=M_CH)
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
    cores = int(os.environ.get("OMP_NUM_THREADS", os.cpu_count() or 1))
    desc = f"{steps} steps x oracle encode+decode of a {W}x{rows} strip ({rows}/{padded(H, W, hyper)[0]} of a padded frame)"
    line = {"impl": "reference", "metric": f"{W}x{H} encode+decode frames/s", "value": round(v, 6),
            "unit": "frames/s", "n_gpus": world, "steps": steps, "warmup": warm, "ms_per_step": round(dt / steps * 1e3, 3),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64 accumulate / f32",
            "data": "synthetic", "config": {"workload": WORKLOAD + " (oracle, bounded strip sample per step)"},
            "cpu_baseline": {"value": round(v, 6), "unit": "frames/s", "cores": cores, "kind": "oracle", "sample": desc},
            "e2e": {"value": round(v, 6), "unit": "frames/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
