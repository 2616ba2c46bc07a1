"""Per-tile timeline of one GEMM-engine layer (CTA 0) at the bench workload.

    python scripts/trace_layer.py gs3 [batch]
Prints, per tile, cycles (relative to the first MMA start) of: producer start, MMA start,
MMA end, norm issue, epilogue start, x^2 written, norm ready, epilogue end.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

from lic_synth import ModelSpec, generate_weights, synth_frames_u8, write_licw
from paper_2208_01641_b200 import lic

layer = sys.argv[1] if len(sys.argv) > 1 else "gs3"
B = int(sys.argv[2]) if len(sys.argv) > 2 else 4
spec = ModelSpec(kind=1, N=128, M=192)
c = lic.Codec(write_licw(spec, generate_weights(spec, 0)), 720, 1280, max_batch=B)
# the real encode + decode path (activation outputs only, no f32 test copies)
frames = synth_frames_u8(B, 720, 1280, seed=3)
ys = np.empty((B,) + c.y_shape, np.int8)
yi = np.empty((B,) + c.y_shape, np.uint8)
zs = np.empty((B,) + c.z_shape, np.int8)
dec = np.empty((B, 720, 1280, 3), np.uint8)


def step():
    c.encode(frames, ys, yi, zs, u8=True)
    if not layer.startswith(("ga", "ha")):
        c.decode(ys, dec, u8=True)


step()
c.trace(layer, True)
step()
t = c.trace_read().astype(np.int64)
names = ["mma_s", "mma_e", "norm_i", "epi_s", "epi_x2", "epi_n", "epi_e", "prod_s"]
bnames = ["b_patch", "b_c0_rdy", "b_c0_done", "b_c1_rdy", "b_c1_done", "mma_k0", "mma_kl", "peerB", "b_raw", "epi_p2", "epi_acq", "epi_stg", "w_halo", "w_b", "b_rawiss", "cta"]
n = int((t[:, 0] > 0).sum())
t0 = t[0, 0]
fused = True
cols = names + (bnames if fused else [])
print(f"{layer}: {n} tiles traced on CTA 0")
print("tile " + " ".join(f"{x:>9s}" for x in cols) + "   mma_dur epi_dur  gap(mma_s[i]-mma_e[i-1])")
for i in range(min(n, 40)):
    row = [(v if name.startswith("w_") else v - t0) if v else -1 for name, v in zip(cols, t[i, :len(cols)])]
    gap = t[i, 0] - t[i - 1, 1] if i else 0
    print(f"{i:4d} " + " ".join(f"{v:9d}" for v in row) + f"   {t[i,1]-t[i,0]:7d} {t[i,6]-t[i,3]:7d} {gap:7d}")
# kernel-relative view: CTA entry (tile slot 0 of "cta"), setup done (slot 1), then tile 0's events
ent, setup = int(t[0, 23]), int(t[1, 23])
if ent:
    print(f"CTA 0: setup {setup - ent} cycles after entry; tile 0 (from entry): producer {t[0,7]-ent}, "
          f"MMA start {t[0,0]-ent}, first operands {t[0,13]-ent}, MMA end {t[0,1]-ent}, epilogue start {t[0,3]-ent}, "
          f"epilogue end {t[0,6]-ent}; last tile epilogue end {t[n-1,6]-ent}")
per_tile = (t[n - 1, 6] - t[0, 0]) / max(n, 1)
print(f"mean cycles per tile (first MMA start -> last epilogue end): {per_tile:.0f}")
print(f"mean MMA-busy per tile: {np.mean(t[:n,1]-t[:n,0]):.0f}, mean epilogue per tile: {np.mean(t[:n,6]-t[:n,3]):.0f}")

