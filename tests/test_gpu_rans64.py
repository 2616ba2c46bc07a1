"""rans64 + bypass on real codec planes (-m gpu): the GPU encoder's 720p y symbols and CDF
indexes (bench workload C3) coded with CompressAI-style Gaussian tables on the codec's
scale table (R23) -- lossless round trip, and with saturated values injected
(escapes) product bytes equal the oracle's."""
import numpy as np
import pytest

from lic_synth import ModelSpec, generate_weights, synth_frames_u8, write_licw
from oracle import rans64 as O
from paper_2208_01641_b200 import lic

pytestmark = pytest.mark.gpu


def test_rans64_on_gpu_planes_720p():
    spec = ModelSpec(kind=1, N=128, M=192)
    w = generate_weights(spec, seed=0)
    c = lic.Codec(write_licw(spec, w), 720, 1280, max_batch=1, device=0)
    fr = synth_frames_u8(1, 720, 1280, seed=11)
    ys = np.empty((1,) + c.y_shape, np.int8)
    yi = np.empty((1,) + c.y_shape, np.uint8)
    zs = np.empty((1,) + c.z_shape, np.int8)
    c.encode(fr, ys, yi, zs, u8=True)
    G = lic.Rans64Tables.gaussian(w["scale_table"])
    sym, idx = ys[0].astype(np.int32).ravel(), yi[0].astype(np.int32).ravel()
    b = G.encode(sym, idx)
    assert (G.decode(b, idx) == sym).all()
    # the codec's planes stay inside the tables (tail mass 1e-9); force the escape path on
    # a few hundred positions with the clamp's extremes (+-L, the values a saturated
    # quantiser writes) and check the whole plane bit-exactly against the oracle
    rng = np.random.default_rng(5)
    pos = rng.choice(sym.size, 300, replace=False)
    sym[pos] = np.where(rng.random(300) < 0.5, -32, 32)
    v = sym - G.offsets[idx]
    assert int(((v < 0) | (v >= G.sizes[idx] - 2)).sum()) > 0
    b = G.encode(sym, idx)
    assert (G.decode(b, idx) == sym).all()
    assert b == O.rans64_encode(sym, idx, G.cdfs, G.sizes, G.offsets)
