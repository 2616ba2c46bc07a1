"""Tiny encode + decode through the C ABI for compute-sanitizer runs:

    compute-sanitizer --tool memcheck python scripts/sanitize.py
Hyperprior 128/192 and factorized at 128 x 192 (f32 and u8 frames), batch 2, GDN and 1DN."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

from lic_synth import ModelSpec, generate_weights, synth_frames_u8, u8_to_f32_chw, write_licw
from paper_2208_01641_b200 import lic

H, W, B = 128, 192, 2
for kind, act in ((1, 0), (0, 0), (0, 1)):
    spec = ModelSpec(kind=kind, N=128, M=192, activation=act)
    c = lic.Codec(write_licw(spec, generate_weights(spec, seed=0)), H, W, max_batch=B, device=0)
    fr = synth_frames_u8(B, H, W, seed=5)
    ys = np.empty((B,) + c.y_shape, np.int8)
    yi = np.empty((B,) + c.y_shape, np.uint8) if kind == 1 else None
    zs = np.empty((B,) + c.z_shape, np.int8) if kind == 1 else None
    c.encode(u8_to_f32_chw(fr), ys, yi, zs)
    c.encode(fr, ys, yi, zs, u8=True)
    if kind == 1:
        c.hyper_indexes(zs, yi)
    out = np.empty((B, H, W, 3), np.uint8)
    c.decode(ys, out, u8=True)
    print(f"kind {kind} act {act}: ok, {int((ys != 0).sum())} nonzero symbols")
