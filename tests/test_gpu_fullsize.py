"""Full-size parity in the bench's launch configuration (-m gpu).

BASELINE.json configs at their real sizes (C3: 1280x720 -> 1280x768, batch 4 as bench.py
times it; C4/C5 shapes for the N=192/M=320 model) are too large for the oracle to run
whole, so every layer is fed seeded random full-size inputs (channel statistics of the
codec's activations) through lic_test_layer and the oracle recomputes SAMPLED output
patches exactly: an output patch of a conv / transposed conv depends only on a bounded
input window, which the oracle evaluates with the zero padding made explicit.  Patches
cover the four corners, the padded edges and random interior tiles of every frame.
"""
import numpy as np
import pytest

from lic_synth import ModelSpec, generate_weights, write_licw
from oracle import oracle as O

from parity import check_float

pytestmark = pytest.mark.gpu

# layer -> (kind, k, stride, activation, weight prefix)
LAYERS = {
    "ga1": ("conv", 5, 2, "gdn"), "ga2": ("conv", 5, 2, "gdn"), "ga3": ("conv", 5, 2, "gdn"),
    "ga4": ("conv", 5, 2, None), "ha1": ("conv", 3, 1, "relu"), "ha2": ("conv", 5, 2, "relu"),
    "ha3": ("conv", 5, 2, None), "hs1": ("deconv", 5, 2, "relu"), "hs2": ("deconv", 5, 2, "relu"),
    "hs3": ("conv", 3, 1, "relu"), "gs1": ("deconv", 5, 2, "igdn"), "gs2": ("deconv", 5, 2, "igdn"),
    "gs3": ("deconv", 5, 2, "igdn"), "gs4": ("deconv", 5, 2, "clip"),
}


def oracle_patch(x, w, layer, oy0, ox0, oh, ow):
    """Oracle output rows [oy0, oy0+oh) x cols [ox0, ox0+ow) of `layer` on input x (C,H,W)."""
    kind, k, s, act = LAYERS[layer]
    C, H, W = x.shape
    p = k // 2
    if kind == "conv":
        iy0, ix0 = s * oy0 - p, s * ox0 - p
        ih, iw = s * (oh - 1) + k, s * (ow - 1) + k
    else:  # transposed conv, stride 2, p 2, output_padding 1: out oy uses in (oy+2-ky)/2
        iy0, ix0 = oy0 // 2 - 1, ox0 // 2 - 1
        ih, iw = (oy0 + oh - 1) // 2 + 2 - iy0, (ox0 + ow - 1) // 2 + 2 - ix0
    win = np.zeros((C, ih, iw), np.float32)
    ys, xs = max(iy0, 0), max(ix0, 0)
    ye, xe = min(iy0 + ih, H), min(ix0 + iw, W)
    win[:, ys - iy0:ye - iy0, xs - ix0:xe - ix0] = x[:, ys:ye, xs:xe]
    if kind == "conv":
        out = O.conv2d(win, w[f"{layer}.w"], w[f"{layer}.b"], s, 0)[:, :oh, :ow]
    else:
        full = O.deconv2d(win, w[f"{layer}.w"], w[f"{layer}.b"], 2, 2, 1)   # rows 2*iy0 ...
        r0, c0 = oy0 - 2 * iy0, ox0 - 2 * ix0
        # rows that depend on inputs outside the window are not used
        out = full[:, r0:r0 + oh, c0:c0 + ow]
    if act == "gdn":
        out = O.gdn(out, w[f"{layer}.beta"], w[f"{layer}.gamma"])
    elif act == "igdn":
        out = O.gdn(out, w[f"{layer}.beta"], w[f"{layer}.gamma"], inverse=True)
    elif act == "relu":
        out = O.relu(out)
    elif act == "clip":
        out = np.clip(out, 0, 1)
    return out


def sample_rects(H, W, rng, n_interior=3, size=(6, 10)):
    h, w = size
    rects = [(0, 0), (0, W - w), (H - h, 0), (H - h, W - w), (H // 2, 0), (0, W // 2)]
    for _ in range(n_interior):
        rects.append((int(rng.integers(0, H - h)), int(rng.integers(0, W - w))))
    return [(y, x, h, w) for y, x in rects]


def input_stats(layer):
    """Rough value scale of each layer's input in the real codec (keeps GDN/IGDN in range)."""
    return {"ga1": ("unif", 1.0), "ha1": ("abs", 0.6), "hs1": ("int", 1.0), "gs1": ("int", 1.5)}.get(
        layer, ("normal", 0.5))


def make_input(shape, layer, rng):
    kind, sc = input_stats(layer)
    if kind == "unif":
        return rng.random(shape, dtype=np.float32)
    if kind == "abs":
        return np.abs(rng.standard_normal(shape).astype(np.float32)) * sc
    if kind == "int":
        return np.clip(np.round(rng.standard_normal(shape) * sc), -32, 32).astype(np.float32)
    return (rng.standard_normal(shape) * sc).astype(np.float32)


def run_layers(spec, H, W, batch, layers, seed=7):
    from paper_2208_01641_b200 import lic
    w = generate_weights(spec, seed=0)
    c = lic.Codec(write_licw(spec, w), H, W, max_batch=batch)
    rng = np.random.default_rng(seed)
    worst = {}
    for layer in layers:
        (ci, hi, wi), (co, ho, wo) = c.layer_shapes(layer)
        x = make_input((batch, ci, hi, wi), layer, rng)
        got = c.test_layer(layer, x)
        assert got.shape == (batch, co, ho, wo)
        err = 0.0
        for b in range(batch):
            for (oy, ox, oh, ow) in sample_rects(ho, wo, rng):
                ref = oracle_patch(x[b], w, layer, oy, ox, oh, ow)
                err = max(err, check_float(got[b, :, oy:oy + oh, ox:ox + ow], ref, what=f"{layer} b{b} @({oy},{ox})"))
        worst[layer] = err
    c.close()
    return worst


@pytest.mark.parametrize("layer", list(LAYERS))
def test_c3_fullsize_layer(layer):
    """configs[2]: hyper N=128 M=192 at 1280x720 (padded 1280x768), batch 4 = bench.py's step."""
    worst = run_layers(ModelSpec(kind=1, N=128, M=192), 720, 1280, 4, [layer])
    print(f"C3 {layer}: max-abs {worst[layer]:.2e}")


@pytest.mark.parametrize("layer", list(LAYERS))
def test_c4_fullsize_layer(layer):
    """configs[3]: hyper N=192 M=320 at 1280x720 (GDN with 192 channels, Cout=320 split over two
    N tiles, Cin=320 layers on the per-tap path)."""
    worst = run_layers(ModelSpec(kind=1, N=192, M=320), 720, 1280, 1, [layer], seed=11)
    print(f"C4 {layer}: max-abs {worst[layer]:.2e}")


def test_c5_geometry_layers():
    """configs[4]: 1920x1080 -> 1920x1088 (odd pad 8: top 4), N=192 M=320, the layers whose
    tile grids differ most from C4."""
    worst = run_layers(ModelSpec(kind=1, N=192, M=320), 1080, 1920, 1, ["ga1", "ga4", "ha3", "gs3", "gs4"],
                       seed=13)
    print("C5", {k: f"{v:.1e}" for k, v in worst.items()})


def test_c2_factorized_layers():
    """configs[1]: factorized N=128 M=192 at 768x512 (no padding)."""
    worst = run_layers(ModelSpec(kind=0, N=128, M=192), 512, 768, 1,
                       ["ga1", "ga2", "ga3", "ga4", "gs1", "gs2", "gs3", "gs4"], seed=17)
    print("C2", {k: f"{v:.1e}" for k, v in worst.items()})
