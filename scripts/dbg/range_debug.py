"""Debug: which g_s layer saturates on the +-4 (seed 12) plane, and how far from the oracle."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
from lic_synth import ModelSpec, generate_weights, write_licw
from oracle import oracle as O
from paper_2208_01641_b200 import lic
spec = ModelSpec(kind=1, N=128, M=192)
w = generate_weights(spec, seed=0)
H, W = 128, 192
c = lic.Codec(write_licw(spec, w), H, W)
ys = np.random.default_rng(12).choice(np.array([-4, 4], np.int8), size=(1,) + c.y_shape).astype(np.int8)
g = ys[0].astype(np.float32)
for i in (1, 2, 3):
    pre = O.deconv2d(g, w[f"gs{i}.w"], w[f"gs{i}.b"], 2, 2, 1)
    ref = O.gdn(pre, w[f"gs{i}.beta"], w[f"gs{i}.gamma"], inverse=True)
    c.range_count(reset=True)
    got = c.test_layer(f"gs{i}", g[None])[0]
    n = c.range_count()
    err = np.abs(got.astype(np.float64) - ref)
    k = np.unravel_index(err.argmax(), err.shape)
    print(f"gs{i}: range {n}, pre max {np.abs(pre).max():.1f}, ref max {np.abs(ref).max():.1f}, got max {np.abs(got).max():.1f}, "
          f"max err {err.max():.3e} at {k} (ref {ref[k]:.3f}, got {got[k]:.3f}, pre {pre[k]:.3f}), normwise {err.max()/np.abs(ref).max():.2e}", flush=True)
    big = np.argwhere(np.abs(got) > 65504)
    print("  |got| > 65504 at", big[:5].tolist(), flush=True)
    g = ref
c.range_count(reset=True)
out = np.empty((1, 3, H, W), np.float32)
c.decode(ys, out)
print("decode range", c.range_count())
ref = O.decode_frame(ys[0], w, True, O.pad_offsets(H, W, True)[2:], H, W)
print("x-hat err", float(np.abs(out[0] - ref).max()))
