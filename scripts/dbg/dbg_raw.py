import os, sys, numpy as np
sys.path.insert(0, '.')
from lic_synth import ModelSpec, generate_weights, synth_frames_u8, write_licw
from paper_2208_01641_b200 import lic
H, W = int(sys.argv[1]), int(sys.argv[2]); B = int(sys.argv[3])
spec = ModelSpec(kind=1, N=128, M=192)
c = lic.Codec(write_licw(spec, generate_weights(spec, 0)), H, W, max_batch=B)
fr = synth_frames_u8(B, H, W, seed=3)
ys = np.empty((B,) + c.y_shape, np.int8); yi = np.empty((B,) + c.y_shape, np.uint8); zs = np.empty((B,) + c.z_shape, np.int8)
c.encode(fr, ys, yi, zs, u8=True)
print("ok", H, W, B, int(ys.astype(np.int64).sum()))
