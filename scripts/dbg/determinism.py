"""Encode-side vs decode-side (hyper_indexes) CDF indexes over repeated runs at C3 (1280x720,
batch 4): they must be identical every time (the coder needs the same tables on both sides)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from lic_synth import ModelSpec, generate_weights, synth_frames_u8, write_licw
from paper_2208_01641_b200 import lic

B, H, W = 4, 720, 1280
n = int(sys.argv[1]) if len(sys.argv) > 1 else 50
spec = ModelSpec(kind=1, N=128, M=192)
c = lic.Codec(write_licw(spec, generate_weights(spec, 0)), H, W, max_batch=B)
bad = 0
ref = None
for i in range(n):
    fr = torch.from_numpy(synth_frames_u8(B, H, W, seed=3 + (i % 3))).cuda()
    ys = torch.empty((B,) + c.y_shape, dtype=torch.int8, device="cuda")
    yi = torch.empty((B,) + c.y_shape, dtype=torch.uint8, device="cuda")
    zs = torch.empty((B,) + c.z_shape, dtype=torch.int8, device="cuda")
    yi2 = torch.empty_like(yi)
    c.encode(fr, ys, yi, zs, u8=True)
    c.hyper_indexes(zs, yi2)
    torch.cuda.synchronize()
    if not torch.equal(yi, yi2):
        bad += 1
        print("mismatch run", i, int((yi != yi2).sum()))
print(f"{n} runs, {bad} encode/decode index mismatches")
