"""Chained full-size parity at the headline configuration (-m gpu).

BASELINE.json configs[2] (C3): scale hyperprior N=128 M=192 on 1280x720 frames (padded to
1280x768), batch 4, u8 frames from HBM -- exactly the launch plan bench.py times
(lic_encode_u8 / lic_hyper_indexes / lic_decode_u8 on a max_batch-4 codec, and the native
pipeline with 32 y substreams).  The oracle runs every frame whole (PAPER.md:72-76
hyperprior encoder / decoder on the 1280x720 workload of PAPER.md:155; ~30 s per frame on
the GPU box's host cores), and the CUDA path is compared stage-wise on identical inputs
(SURVEY.md §8(c) c17):

  * encode: y and z (fp32 debug copies) within 1e-3, y / z symbols with the tie rule,
    y indexes with the boundary rule (c18) -- against the oracle's h_s on the oracle's z, or,
    where a z symbol flipped at a tie, on the GPU's z (the indexes follow z-hat, c17);
  * decoder GPU1 from the oracle's z symbols: indexes with the boundary rule;
  * decoder GPU2 from the oracle's y symbols: x-hat within 1e-3 (f32), +-1 (u8);
  * bitstreams (c19): every pipeline string equals the oracle coder run on the GPU's planes
    byte for byte (i) and decodes losslessly with the oracle decoder (iii); a frame whose
    planes equal the oracle's has exactly the oracle's strings (ii).  Frames whose planes
    differ are COUNTED and reported, and every differing symbol / index must be a legal
    c18 tie: at 1280x720 about 1e-5 of the y symbols lie within the split-FP16 rounding
    error (~1e-6) of a .5 tie, so a frame with a flipped symbol is expected now and then
    (R19).

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


def _check_frame(r, w, ys, yi, zs, what):
    """c18 on one frame's GPU planes.  Returns (y flips, z flips, index flips)."""
    nz = check_symbols(zs, r["z_sym"], r["z"] - w["mu_z"][:, None, None], what=f"{what} z_sym")
    ny = check_symbols(ys, r["y_sym"], r["y"], what=f"{what} y_sym")
    if nz == 0:
        sig, idx = r["sigma"], r["y_idx"]
    else:                                   # the indexes follow the GPU's z-hat
        sig = O.h_s(O.dequantize(zs, w["mu_z"]), w)
        idx = O.scale_index(sig, w["scale_table"])
    ni = check_indexes(yi, idx, sig, w["scale_table"], what=f"{what} y_idx")
    return ny, nz, ni


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
    w = c3["w"]
    assert abs(int(nsat) - sum(int(r["n_sat"]) for r in c3["ref"])) <= 1
    n_sym = n_idx = 0
    for b, r in enumerate(c3["ref"]):
        ey = check_float(y[b], r["y"], what=f"C3 y frame {b}")
        ez = check_float(z[b], r["z"], what=f"C3 z frame {b}")
        ny, nz, ni = _check_frame(r, w, ys[b], yi[b], zs[b], f"C3 frame {b}")
        if nz == 0:
            check_float(sig[b], r["sigma"], what=f"C3 sigma {b}")
        n_sym += ny + nz
        n_idx += ni
        print(f"C3 frame {b}: y {ey:.2e}, z {ez:.2e}, y_sym off {ny}, z_sym off {nz}, y_idx off {ni}")
    print(f"C3 batch {B}: {n_sym} symbol and {n_idx} index flips (all at c18 ties) over {B} frames")


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


@pytest.mark.parametrize("parts", [2, 1])
def test_c3_pipeline_bitstreams_bit_exact(lic, codec, c3, parts):
    """c19 through the bench's own pipeline (batch 4, 32 y substreams, frames in HBM; each frame's
    y string coded as 2 slab ranges on separate coder threads as bench.py runs it, or as 1)."""
    import torch
    dev_in = torch.from_numpy(c3["frames"]).cuda()
    dev_out = torch.empty_like(dev_in)
    ys, yi, zs, _ = _encode(codec, dev_in, B)          # the planes the pipeline codes (deterministic)
    pipe = lic.Pipeline(codec, coder_threads=4, batch=B, inflight=2, u8=True, keep_bitstreams=True,
                        substreams=K_SUB, coder_parts=parts)
    st = pipe.run(dev_in, dev_out, B)
    assert st["symbol_mismatches"] == 0
    tabs, w = c3["tabs"], c3["w"]
    differ = []
    for b, r in enumerate(c3["ref"]):
        yb, zb = pipe.bitstream(b)
        zrows = O.channel_rows(zs[b].shape)
        # (i) the pipeline's strings are the oracle coder's strings of the GPU's planes
        assert yb == O.rans_encode_slabs(ys[b], yi[b], tabs.gauss, K_SUB)
        assert zb == O.rans_encode(zs[b], zrows, tabs.z)
        # (iii) and decode losslessly with the oracle decoder (GPU1's indexes, as the decoder has)
        zd = O.rans_decode(zb, zrows, tabs.z).reshape(zs[b].shape)
        yd = O.rans_decode_slabs(yb, ys[b].shape, yi[b], tabs.gauss, K_SUB)
        assert np.array_equal(yd, ys[b]) and np.array_equal(zd, zs[b])
        # (ii) identical planes -> the oracle's own strings; otherwise counted, ties only
        same = (np.array_equal(ys[b], r["y_sym"]) and np.array_equal(yi[b], r["y_idx"])
                and np.array_equal(zs[b], r["z_sym"]))
        if same:
            assert yb == O.rans_encode_slabs(r["y_sym"], r["y_idx"], tabs.gauss, K_SUB)
            assert zb == O.rans_encode(r["z_sym"], zrows, tabs.z)
        else:
            differ.append((b,) + _check_frame(r, w, ys[b], yi[b], zs[b], f"C3 pipeline frame {b}"))
    pipe.close()
    print(f"C3 pipeline: {B - len(differ)} of {B} frames bit-exact with the oracle's bitstreams; "
          f"frames with tie flips (frame, y, z, idx): {differ}")
    # the pipeline's decoded frames against the oracle's decode of the same (GPU) symbols --
    # one frame (the oracle decoder takes ~25 s per 720p frame); x-hat of flipped symbols
    # differs from the oracle-symbol x-hat by design (c17), so the oracle decodes ys[1]
    out = dev_out.cpu().numpy()
    ref1 = O.decode_frame(ys[1], w, True, O.pad_offsets(H, W, True)[2:], H, W)
    ref8 = np.floor(np.moveaxis(ref1, 0, -1).astype(np.float64) * 255 + 0.5)
    assert np.max(np.abs(out[1].astype(np.int32) - ref8)) <= 1


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
    ny, nz, ni = _check_frame(r, w, ys[0], yi[0], zs[0], "C4")
    yi2 = np.empty_like(yi)
    c.hyper_indexes(r["z_sym"][None], yi2)
    check_indexes(yi2[0], r["y_idx"], r["sigma"], w["scale_table"], what="C4 GPU1")
    out = np.empty((1, 3, H, W), np.float32)
    c.decode(r["y_sym"][None], out)
    ex = check_float(out[0], r["xhat"], what="C4 x-hat")
    tabs = O.build_tables(w, True, 32)
    # c19 (i): product coder on the GPU planes == oracle coder on the same planes
    gpu = {"y_sym": ys[0], "y_idx": yi[0], "z_sym": zs[0]}
    yb_ref, zb_ref = O.code_planes(gpu, tabs, True)
    yb = lic.rans_encode(ys[0].ravel(), c.cdf(2), rows=yi[0].ravel())
    assert yb == yb_ref and lic.rans_encode(zs[0], c.cdf(1)) == zb_ref
    assert np.array_equal(O.rans_decode(yb, yi[0].astype(np.int32), tabs.gauss).reshape(ys[0].shape), ys[0])
    print(f"C4: y_sym flips {ny}, z_sym flips {nz}, y_idx flips {ni} (all at c18 ties), x-hat max-abs {ex:.2e}")
    c.close()
