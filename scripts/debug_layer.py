"""Debug helper: one layer through lic_test_layer vs the oracle on a small random input,
error statistics by sub-pixel phase and tile position (GPU box)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

from lic_synth import ModelSpec, generate_weights, write_licw
from oracle import oracle as O
from paper_2208_01641_b200 import lic

layer = sys.argv[1] if len(sys.argv) > 1 else "gs4"
H, W = int(sys.argv[2]) if len(sys.argv) > 2 else 128, int(sys.argv[3]) if len(sys.argv) > 3 else 192
spec = ModelSpec(kind=1, N=128, M=192)
w = generate_weights(spec, 0)
c = lic.Codec(write_licw(spec, w), H, W, max_batch=1)
shp_in, shp_out = c.layer_shapes(layer)
rng = np.random.default_rng(0)
x = (rng.standard_normal((1,) + tuple(shp_in)) * 0.5).astype(np.float32)
got = c.test_layer(layer, x)[0]
ref = np.clip(O.deconv2d(x[0], w["gs4.w"], w["gs4.b"], 2, 2, 1), 0, 1)
err = np.abs(got - ref)
print("shape", got.shape, "max err", err.max(), "frac bad", (err > 1e-3).mean())
for py in range(2):
    for px in range(2):
        e = err[:, py::2, px::2]
        print(f"phase ({py},{px}): max {e.max():.3e} bad {(e > 1e-3).mean():.3f}")
gy = np.arange(got.shape[1]) // 2
gx = np.arange(got.shape[2]) // 2
bad = (err.max(0) > 1e-3)
print("bad by grid x mod 14:", [round(bad[:, (gx % 14) == k].mean(), 3) for k in range(14)])
print("bad by grid y mod 6:", [round(bad[(gy % 6) == k, :].mean(), 3) for k in range(6)])
print("bad by channel:", [round((err[ch] > 1e-3).mean(), 3) for ch in range(3)])
print("sample got/ref:", got[:, 4, 6], ref[:, 4, 6])
