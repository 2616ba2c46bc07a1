"""Debug: run each layer through lic_test_layer in LIC_PREC_F16, one process per layer."""
import os, subprocess, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
LAYERS = ["ga1", "ga2", "ga3", "ga4", "gs1", "gs2", "gs3", "gs4", "ha1", "ha2", "ha3", "hs1", "hs2", "hs3"]
code = '''
import sys, numpy as np
sys.path.insert(0, ".")
from lic_synth import ModelSpec, generate_weights, write_licw
from paper_2208_01641_b200 import lic
spec = ModelSpec(kind=1, N=128, M=192)
c = lic.Codec(write_licw(spec, generate_weights(spec, 0)), 240, 300, max_batch=1, precision=int(sys.argv[2]))
i, o = c.layer_shapes(sys.argv[1])
x = np.random.default_rng(0).standard_normal((1,) + i).astype(np.float32) * 0.3
try:
    c.test_layer(sys.argv[1], x); print(sys.argv[1], "ok")
except Exception as e:
    print(sys.argv[1], "FAIL", e)
'''
for L in LAYERS:
    r = subprocess.run([sys.executable, "-c", code, L, sys.argv[1] if len(sys.argv) > 1 else "1"], capture_output=True, text=True)
    print((r.stdout + r.stderr).strip().splitlines()[-1])
