"""Debug: does any kernel read workspace memory it did not write?  Fill a bound workspace with
0xFF (fp16 NaN) or 0x7B (fp16 ~6e4) and compare encode/decode with a zero-filled one."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import torch
from lic_synth import ModelSpec, generate_weights, write_licw, synth_frames_u8
from paper_2208_01641_b200 import lic
spec = ModelSpec(kind=1, N=128, M=192)
w = generate_weights(spec, seed=0)
for (H, W, B) in ((128, 192, 1), (136, 200, 2), (720, 1280, 4)):
    c = lic.Codec(write_licw(spec, w), H, W, max_batch=B)
    ys = np.random.default_rng(12).choice(np.array([-4, 4], np.int8), size=(B,) + c.y_shape).astype(np.int8)
    fr = synth_frames_u8(B, H, W, seed=3)
    res = {}
    for fill in (0x00, 0xFF, 0x7B):
        ws = torch.full((c.workspace_bytes(),), fill, dtype=torch.uint8, device="cuda")
        c.bind_workspace(ws)
        c.range_count(reset=True)
        out = np.empty((B, 3, H, W), np.float32)
        c.decode(ys, out)
        r1 = c.range_count()
        e_ys = np.empty((B,) + c.y_shape, np.int8); e_yi = np.empty((B,) + c.y_shape, np.uint8); e_zs = np.empty((B,) + c.z_shape, np.int8)
        c.encode(fr, e_ys, e_yi, e_zs, u8=True)
        r2 = c.range_count()
        res[fill] = (out, e_ys, e_yi, e_zs)
        print(f"{H}x{W} b{B} fill {fill:#x}: decode range {r1}, encode range {r2}, finite {np.isfinite(out).all()}", flush=True)
    for fill in (0xFF, 0x7B):
        same = [np.array_equal(a, b) for a, b in zip(res[0], res[fill])]
        print(f"  fill {fill:#x} identical to zero fill (xhat, y_sym, y_idx, z_sym): {same}", flush=True)
        if not same[0]:
            d = np.abs(res[0][0] - res[fill][0]); k = np.argwhere(d > 0)
            print("   xhat differs at", len(k), "samples, first", k[:5].tolist(), flush=True)
    c.close()
