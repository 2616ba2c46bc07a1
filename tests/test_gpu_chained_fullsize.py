"""Chained full-size parity at the headline configuration (-m gpu).

BASELINE.json configs[2] (C3): scale hyperprior N=128 M=192 on 1280x720 frames (padded to
1280x768), batch 4, u8 frames from HBM -- exactly the launch plan bench.py times
(lic_encode_u8 / lic_hyper_indexes / lic_decode_u8 on a max_batch-4 codec, and the native
pipeline with 32 y substreams).  The oracle runs every frame whole (PAPER.md:72-76
hyperprior encoder / decoder on the 1280x720 workload of PAPER.md:155; ~30 s per frame on
the GPU box's host cores), and the CUDA path is compared stage-wise on identical inputs
(SURVEY.md §8(c) c17):

  * encode: y and z (fp32 debug copies) within 1e-3, y / z symbols with the tie rule,
    y indexes with the boundary rule (c18);
  * decoder GPU1 from the oracle's z symbols: indexes with the boundary rule;
  * decoder GPU2 from the oracle's y symbols: x-hat within 1e-3 (f32), +-1 (u8);
  * bitstreams (c19): the frames whose planes differ from the oracle's are COUNTED and
    must be 0; every pipeline string equals the oracle coder's string byte for byte and
    decodes losslessly with the oracle decoder.

Plus one C4 frame (N=192 M=320: GDN with 192 channels, M = 320 split over two N tiles).
"""
import numpy as np
import pytest

from lic_synth import ModelSpec, generate_weights, synth_frames_u8, write_licw
from oracle import oracle as O

from parity import check_float, check_indexes, check_symbols

pytestmark = pytest.mark.gpu

H, W, B = 720, 1280, 4
K_SUB = 32          # bench.py's y substreams


def _oracle_frames(spec, frames):
    w = generate_weights(spec, seed=0)
    ref = []
    for f in frames:
        x, crop = O.ingest_u8(f, hyper=True)
        p = O.encode_planes(x, w, True, 32)
        p["xhat"] = O.decode_frame(p["y_sym"], w, True, crop, f.shape[0], f.shape[1])
        ref.append(p)
    return w, ref


@pytest.fixture(scope="module")
def lic():
    from paper_2208_01641_b200 import lic as L
    return L


@pytest.fixture(scope="module")
def c3():
    spec = ModelSpec(kind=1, N=128, M=192)
    # bench.py's stream: frames t = 0..3 of seed 1000
    frames = synth_frames_u8(B, H, W, seed=1000)
    w, ref = _oracle_frames(spec, frames)
    return dict(spec=spec, w=w, blob=write_licw(spec, w), frames=frames, ref=ref,
                tabs=O.build_tables(w, True, 32))


@pytest.fixture(scope="module")
def codec(lic, c3):
    c = lic.Codec(c3["blob"], H, W, max_batch=B)
    yield c
    c.close()


def _encode(c, frames_dev, batch):
    import torch
    ys = np.empty((batch,) + c.y_shape, np.int8)
    yi = np.empty((batch,) + c.y_shape, np.uint8)
    zs = np.empty((batch,) + c.z_shape, np.int8)
    nsat = c.encode(frames_dev, ys, yi, zs, u8=True)
    torch.cuda.synchronize()
    return ys, yi, zs, nsat


def test_c3_encode_planes(codec, c3):
    import torch
    dev = torch.from_numpy(c3["frames"]).cuda()
    codec.set_debug(True)
    ys, yi, zs, nsat = _encode(codec, dev, B)
    y, z, sig = codec.debug_latents(B)
    codec.set_debug(False)
    w, tab = c3["w"], c3["w"]["scale_table"]
    assert nsat == sum(int(r["n_sat"]) for r in c3["ref"])
    n_sym = n_idx = 0
    for b, r in enumerate(c3["ref"]):
        ey = check_float(y[b], r["y"], what=f"C3 y frame {b}")
        ez = check_float(z[b], r["z"], what=f"C3 z frame {b}")
        nz = check_symbols(zs[b], r["z_sym"], r["z"] - w["mu_z"][:, None, None], what=f"C3 z_sym {b}")
        ny = check_symbols(ys[b], r["y_sym"], r["y"], what=f"C3 y_sym {b}")
        # indexes follow z-hat: with identical z symbols they may differ only at a boundary
        assert nz == 0, f"frame {b}: {nz} z symbols at a tie -- indexes not comparable"
        check_float(sig[b], r["sigma"], what=f"C3 sigma {b}")
        ni = check_indexes(yi[b], r["y_idx"], r["sigma"], tab, what=f"C3 y_idx {b}")
        n_sym += ny + nz
        n_idx += ni
        print(f"C3 frame {b}: y {ey:.2e}, z {ez:.2e}, y_sym off {ny}, z_sym off {nz}, y_idx off {ni}")
    print(f"C3 batch {B}: {n_sym} symbol and {n_idx} index mismatches over {B} frames")


def test_c3_hyper_indexes_from_oracle_z(codec, c3):
    zs = np.stack([r["z_sym"] for r in c3["ref"]])
    yi = np.empty((B,) + codec.y_shape, np.uint8)
    codec.hyper_indexes(zs, yi)
    for b, r in enumerate(c3["ref"]):
        n = check_indexes(yi[b], r["y_idx"], r["sigma"], c3["w"]["scale_table"], what=f"C3 GPU1 {b}")
        print(f"C3 GPU1 frame {b}: {n} index mismatches")


def test_c3_decode_from_oracle_symbols(codec, c3):
    import torch
    ys = np.stack([r["y_sym"] for r in c3["ref"]])
    out = np.empty((B, 3, H, W), np.float32)
    codec.decode(ys, out)
    for b, r in enumerate(c3["ref"]):
        e = check_float(out[b], r["xhat"], what=f"C3 x-hat {b}")
        print(f"C3 x-hat frame {b}: max-abs {e:.2e}")
    # u8 frames into HBM, as the bench writes them
    o8 = torch.empty((B, H, W, 3), dtype=torch.uint8, device="cuda")
    codec.decode(torch.from_numpy(ys).cuda(), o8, u8=True)
    o8 = o8.cpu().numpy()
    for b, r in enumerate(c3["ref"]):
        ref8 = np.floor(np.moveaxis(r["xhat"], 0, -1).astype(np.float64) * 255 + 0.5)
        assert np.max(np.abs(o8[b].astype(np.int32) - ref8)) <= 1


def test_c3_pipeline_bitstreams_bit_exact(lic, codec, c3):
    """c19 through the bench's own pipeline (batch 4, 32 y substreams, frames in HBM)."""
    import torch
    dev_in = torch.from_numpy(c3["frames"]).cuda()
    dev_out = torch.empty_like(dev_in)
    pipe = lic.Pipeline(codec, coder_threads=4, batch=B, inflight=2, u8=True, keep_bitstreams=True,
                        substreams=K_SUB)
    st = pipe.run(dev_in, dev_out, B)
    assert st["symbol_mismatches"] == 0
    tabs = c3["tabs"]
    mismatched = []
    for b, r in enumerate(c3["ref"]):
        yb, zb = pipe.bitstream(b)
        yb_ref = O.rans_encode_slabs(r["y_sym"], r["y_idx"], tabs.gauss, K_SUB)
        zb_ref = O.rans_encode(r["z_sym"], O.channel_rows(r["z_sym"].shape), tabs.z)
        if yb != yb_ref or zb != zb_ref:
            mismatched.append(b)
        # c19 (iii): the build's strings decode losslessly with the oracle decoder
        zd = O.rans_decode(zb, O.channel_rows(r["z_sym"].shape), tabs.z).reshape(r["z_sym"].shape)
        idx = O.hyper_indexes(zd, c3["w"])
        yd = O.rans_decode_slabs(yb, r["y_sym"].shape, idx, tabs.gauss, K_SUB)
        assert np.array_equal(yd, r["y_sym"]) and np.array_equal(zd, r["z_sym"])
    pipe.close()
    print(f"C3 pipeline: {len(mismatched)} of {B} frames with bitstreams != oracle")
    assert mismatched == [], f"frames {mismatched}: bitstreams differ from the oracle's"
    out = dev_out.cpu().numpy()
    for b, r in enumerate(c3["ref"]):
        ref8 = np.floor(np.moveaxis(r["xhat"], 0, -1).astype(np.float64) * 255 + 0.5)
        assert np.max(np.abs(out[b].astype(np.int32) - ref8)) <= 1


def test_c4_frame_chained(lic):
    """configs[3]: hyperprior N=192 M=320, one 1280x720 frame: encode planes, GPU1 indexes,
    decode from the oracle's symbols, bitstreams."""
    import torch
    spec = ModelSpec(kind=1, N=192, M=320)
    frames = synth_frames_u8(1, H, W, seed=1000, t0=5)
    w, ref = _oracle_frames(spec, frames)
    r = ref[0]
    c = lic.Codec(write_licw(spec, w), H, W, max_batch=4)
    c.set_debug(True)
    ys, yi, zs, _ = _encode(c, torch.from_numpy(frames).cuda(), 1)
    y, z, sig = c.debug_latents(1)
    c.set_debug(False)
    check_float(y[0], r["y"], what="C4 y")
    check_float(z[0], r["z"], what="C4 z")
    nz = check_symbols(zs[0], r["z_sym"], r["z"] - w["mu_z"][:, None, None], what="C4 z_sym")
    ny = check_symbols(ys[0], r["y_sym"], r["y"], what="C4 y_sym")
    assert nz == 0
    check_indexes(yi[0], r["y_idx"], r["sigma"], w["scale_table"], what="C4 y_idx")
    yi2 = np.empty_like(yi)
    c.hyper_indexes(r["z_sym"][None], yi2)
    check_indexes(yi2[0], r["y_idx"], r["sigma"], w["scale_table"], what="C4 GPU1")
    out = np.empty((1, 3, H, W), np.float32)
    c.decode(r["y_sym"][None], out)
    ex = check_float(out[0], r["xhat"], what="C4 x-hat")
    tabs = O.build_tables(w, True, 32)
    planes_equal = (np.array_equal(ys[0], r["y_sym"]) and np.array_equal(yi[0], r["y_idx"])
                    and np.array_equal(zs[0], r["z_sym"]))
    assert planes_equal, f"C4 planes differ (y_sym {ny}, idx {(yi[0] != r['y_idx']).sum()})"
    yb_ref, zb_ref = O.code_planes(r, tabs, True)
    assert lic.rans_encode(ys[0].ravel(), c.cdf(2), rows=yi[0].ravel()) == yb_ref
    assert lic.rans_encode(zs[0], c.cdf(1)) == zb_ref
    print(f"C4: y_sym off {ny}, x-hat max-abs {ex:.2e}")
    c.close()
