"""One warm-up pass + one profiled pass of the full hot path (encode, hyper_indexes,
decode) at the bench workload, in a fixed kernel order for ncu:

  conv_umma launches per pass: ga1 ga2 ga3 ga4 ha1 ha2 ha3 hs1 hs2 hs3 | hs1 hs2 hs3 | gs1 gs2 gs3 gs4
  (plus sym_ingest before each decoder stage; frame ingest is fused into ga1)

    ncu --set full -k regex:conv_umma -s 17 -c 17 -o prof python scripts/profile_step.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch

from lic_synth import ModelSpec, generate_weights, synth_frames_u8, write_licw
from paper_2208_01641_b200 import lic

B = int(os.environ.get("LIC_BATCH", "4"))
H, W = 720, 1280
spec = ModelSpec(kind=1, N=128, M=192)
codec = lic.Codec(write_licw(spec, generate_weights(spec, 0)), H, W, max_batch=B)
fr = torch.from_numpy(synth_frames_u8(B, H, W, seed=3)).cuda()
out = torch.empty_like(fr)
ys = torch.empty((B,) + codec.y_shape, dtype=torch.int8, device="cuda")
yi = torch.empty((B,) + codec.y_shape, dtype=torch.uint8, device="cuda")
zs = torch.empty((B,) + codec.z_shape, dtype=torch.int8, device="cuda")
yi2 = torch.empty_like(yi)
for _ in range(2):
    codec.encode(fr, ys, yi, zs, u8=True)
    codec.hyper_indexes(zs, yi2)
    codec.decode(ys, out, u8=True)
torch.cuda.synchronize()
assert torch.equal(yi, yi2)
print("ok", flush=True)
