"""The streaming pipeline (lic_pipeline_*) on the GPU -- -m gpu.

SPEC.md acceptance #3 (pipelined == serial, bit-identical), latent fidelity (decoded
symbols == encoded), the oracle decodes every string (SURVEY.md c19 iii),
the decoded frames equal a direct lic_decode of the same symbols, and the pinned pool's
reuse / foreign-release semantics.
"""
import numpy as np
import pytest

from lic_synth import ModelSpec, generate_weights, synth_frames_u8, write_licw
from oracle import oracle as O

pytestmark = pytest.mark.gpu

H, W = 200, 300            # pads to 256 x 320 (hyper) / 208 x 304 (factorized)
NF, B = 8, 2


@pytest.fixture(scope="module")
def lic():
    from paper_2208_01641_b200 import lic as L
    return L


def run_pipeline(lic, codec, frames, serial, inflight=3, threads=3, substreams=1, coder=0, parts=1):
    import torch
    fin = torch.from_numpy(frames).cuda()
    fout = torch.zeros_like(fin)
    p = lic.Pipeline(codec, coder_threads=threads, batch=B, inflight=inflight, u8=True, serial=serial,
                     keep_bitstreams=True, substreams=substreams, coder=coder, coder_parts=parts)
    st = p.run(fin, fout, NF)
    streams = [p.bitstream(i) for i in range(NF)]
    p.close()
    return st, streams, fout.cpu().numpy()


@pytest.mark.parametrize("kind,K", [(1, 1), (0, 1), (1, 8), (0, 5)])
def test_pipeline_matches_serial_and_direct(lic, kind, K):
    """K > 1: the y string as K channel-slab substreams (R21), byte-identical to the
    oracle's framing of the same planes."""
    spec = ModelSpec(kind=kind, N=128, M=192)
    w = generate_weights(spec, seed=0)
    codec = lic.Codec(write_licw(spec, w), H, W, max_batch=B)
    frames = synth_frames_u8(NF, H, W, seed=21)
    st, streams, out = run_pipeline(lic, codec, frames, serial=False, substreams=K)
    st_s, streams_s, out_s = run_pipeline(lic, codec, frames, serial=True, substreams=K)
    assert st["frames"] == NF and st["symbol_mismatches"] == 0 and st_s["symbol_mismatches"] == 0
    assert streams == streams_s                               # SPEC.md acceptance #3
    assert np.array_equal(out, out_s)
    # direct path: lic_encode_u8 + the reference (unprepared) host coder
    hyper = kind == 1
    tabs_y = codec.cdf(2 if hyper else 0)
    tabs_z = codec.cdf(1) if hyper else None
    for b0 in range(0, NF, B):
        ys = np.empty((B,) + codec.y_shape, np.int8)
        yi = np.empty((B,) + codec.y_shape, np.uint8) if hyper else None
        zs = np.empty((B,) + codec.z_shape, np.int8) if hyper else None
        codec.encode(np.ascontiguousarray(frames[b0:b0 + B]), ys, yi, zs, u8=True)
        dec = np.empty((B, H, W, 3), np.uint8)
        codec.decode(ys, dec, u8=True)
        assert np.array_equal(dec, out[b0:b0 + B])
        for f in range(B):
            yb, zb = streams[b0 + f]
            if K > 1:
                assert yb == O.rans_encode_slabs(ys[f], yi[f] if hyper else None, tabs_y, K)
                assert np.array_equal(O.rans_decode_slabs(yb, ys[f].shape, yi[f] if hyper else None, tabs_y, K),
                                      ys[f])
                if hyper:
                    assert zb == O.rans_encode(zs[f], O.channel_rows(zs[f].shape), tabs_z)
                continue
            if hyper:
                assert yb == lic.rans_encode(ys[f].ravel(), tabs_y, rows=yi[f].ravel())
                assert zb == lic.rans_encode(zs[f], tabs_z)
                # the oracle decodes the strings (z first, then y with the indexes)
                zd = O.rans_decode(zb, O.channel_rows(zs[f].shape), tabs_z).reshape(zs[f].shape)
                assert np.array_equal(zd, zs[f])
                assert np.array_equal(O.rans_decode(yb, yi[f].astype(np.int32), tabs_y).reshape(ys[f].shape), ys[f])
            else:
                assert zb is None
                assert yb == lic.rans_encode(ys[f], tabs_y)
                assert np.array_equal(O.rans_decode(yb, O.channel_rows(ys[f].shape), tabs_y).reshape(ys[f].shape),
                                      ys[f])
    codec.close()


@pytest.mark.parametrize("kind", [1, 0])
def test_pipeline_rans64_coder(lic, kind):
    """coder = 1: the rans64 + bypass coder (R23) inside the pipeline -- lossless,
    pipelined == serial, every string equal to the direct coder on the GPU planes and, for
    the first frame, to the oracle's."""
    from oracle import rans64 as O64
    spec = ModelSpec(kind=kind, N=128, M=192)
    w = generate_weights(spec, seed=0)
    codec = lic.Codec(write_licw(spec, w), H, W, max_batch=B)
    frames = synth_frames_u8(NF, H, W, seed=23)
    st, streams, out = run_pipeline(lic, codec, frames, serial=False, coder=1)
    st_s, streams_s, out_s = run_pipeline(lic, codec, frames, serial=True, coder=1)
    assert st["frames"] == NF and st["symbol_mismatches"] == 0 and st_s["symbol_mismatches"] == 0
    assert streams == streams_s and np.array_equal(out, out_s)
    hyper = kind == 1
    ty = lic.Rans64Tables.gaussian(codec.sigmas(2 if hyper else 0))
    tz = lic.Rans64Tables.gaussian(codec.sigmas(1)) if hyper else None
    for b0 in range(0, NF, B):
        ys = np.empty((B,) + codec.y_shape, np.int8)
        yi = np.empty((B,) + codec.y_shape, np.uint8) if hyper else None
        zs = np.empty((B,) + codec.z_shape, np.int8) if hyper else None
        codec.encode(np.ascontiguousarray(frames[b0:b0 + B]), ys, yi, zs, u8=True)
        for f in range(B):
            yb, zb = streams[b0 + f]
            ry = yi[f].ravel() if hyper else O.channel_rows(ys[f].shape).ravel()
            assert yb == ty.encode(ys[f].ravel(), ry)
            if hyper:
                rz = O.channel_rows(zs[f].shape).ravel()
                assert zb == tz.encode(zs[f].ravel(), rz)
            if b0 + f == 0:
                assert yb == O64.rans64_encode(ys[f].ravel(), ry, ty.cdfs, ty.sizes, ty.offsets)
                if hyper:
                    assert zb == O64.rans64_encode(zs[f].ravel(), rz, tz.cdfs, tz.sizes, tz.offsets)
    codec.close()


def test_pinned_pool_semantics(lic):
    spec = ModelSpec(kind=0, N=128, M=192)
    codec = lic.Codec(write_licw(spec, generate_weights(spec, 0)), 64, 64)
    a = codec.buf_acquire(4096)
    codec.buf_release(a)
    b = codec.buf_acquire(4096)
    assert a == b                                           # reuse before allocation
    assert codec.buf_stats() == (1, 1)
    c = codec.buf_acquire(8192)
    assert c != b and codec.buf_stats() == (2, 1)
    assert codec.buf_release(12345678) == lic.LIC_EFOREIGN
    codec.buf_release(b)
    codec.buf_release(c)
    for _ in range(100):                                    # steady state: no new allocations
        x = codec.buf_acquire(4096)
        codec.buf_release(x)
    assert codec.buf_stats()[0] == 2
    codec.close()


def test_zero_copy_toggle_same_result(lic):
    """PAPER.md:103 zero-copy option: same symbols through mapped pinned planes."""
    import torch
    spec = ModelSpec(kind=1, N=128, M=192)
    codec = lic.Codec(write_licw(spec, generate_weights(spec, 0)), H, W, max_batch=B)
    fr = np.ascontiguousarray(synth_frames_u8(B, H, W, seed=5))
    outs = []
    for zc in (False, True):
        codec.set_zero_copy(zc)
        ys = torch.empty((B,) + codec.y_shape, dtype=torch.int8).pin_memory()
        yi = torch.empty((B,) + codec.y_shape, dtype=torch.uint8).pin_memory()
        zs = torch.empty((B,) + codec.z_shape, dtype=torch.int8).pin_memory()
        codec.encode(fr, ys, yi, zs, u8=True)
        outs.append((ys.numpy().copy(), yi.numpy().copy(), zs.numpy().copy()))
    for a, b in zip(*outs):
        assert np.array_equal(a, b)
    codec.close()


def test_errors_are_status_codes(lic):
    spec = ModelSpec(kind=1, N=128, M=192)
    codec = lic.Codec(write_licw(spec, generate_weights(spec, 0)), 128, 128, max_batch=1)
    ys = np.empty((2,) + codec.y_shape, np.int8)
    with pytest.raises(lic.LicError) as e:                  # batch > max_batch
        codec.encode(np.zeros((2, 3, 128, 128), np.float32), ys, ys.view(np.uint8), ys)
    assert e.value.status == lic.LIC_ESHAPE
    with pytest.raises(lic.LicError) as e:                  # hyper codec without y_idx / z_sym
        codec.encode(np.zeros((1, 3, 128, 128), np.float32), ys[:1])
    assert e.value.status == lic.LIC_EINVAL
    bad = bytearray(write_licw(spec, generate_weights(spec, 0)))
    with pytest.raises(lic.LicError) as e:                  # truncated weights container
        lic.Codec(bytes(bad[:-10]), 128, 128)
    assert e.value.status == lic.LIC_EDIGEST
    codec.close()


@pytest.mark.parametrize("K,parts", [(32, 2), (32, 4), (16, 2)])
def test_coder_parts_same_bitstreams(lic, K, parts):
    """Each frame's y string coded as `parts` slab ranges on separate coder threads
    (lic_rans_encode_slab_range / lic_rans_decode_slab_range): the same strings, frames and
    lossless round trip as one coder task per frame."""
    spec = ModelSpec(kind=1, N=128, M=192)
    codec = lic.Codec(write_licw(spec, generate_weights(spec, seed=0)), H, W, max_batch=B)
    frames = synth_frames_u8(NF, H, W, seed=23)
    st1, s1, o1 = run_pipeline(lic, codec, frames, serial=False, substreams=K, threads=4, parts=1)
    st2, s2, o2 = run_pipeline(lic, codec, frames, serial=False, substreams=K, threads=4, parts=parts)
    assert st1["symbol_mismatches"] == 0 and st2["symbol_mismatches"] == 0
    assert s1 == s2 and np.array_equal(o1, o2)
    codec.close()
