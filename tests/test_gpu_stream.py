"""Streaming demonstration over loopback TCP (§VI) -- -m gpu.

The paper's demo: factorized-prior + 1DN, 1280x720 at 30 FPS, every frame a keyframe, "no
frame drops or noticeable jittering".  Checked: every sequence arrives
once and in order, the receiver's y symbols equal the sender's bit for bit (latent
fidelity through the network path), decoded frames equal a direct lic_decode of the same
symbols, pacing holds the target rate, a weights-digest mismatch aborts before any frame,
and a corrupted frame is counted while the stream continues.
"""
import numpy as np
import pytest

from lic_synth import ModelSpec, generate_weights, synth_frames_u8, write_licw
from lic_synth.weights import ACT_1DN

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def S():
    from paper_2208_01641_b200 import stream
    return stream


def _blob(kind=0, act=ACT_1DN, seed=0):
    spec = ModelSpec(kind=kind, N=128, M=192, activation=act)
    return write_licw(spec, generate_weights(spec, seed))


def test_paper_demo_720p_30fps(S):
    """factorized + 1DN at 1280x720, 30 FPS, 90 frames (3 s)."""
    H, W, n = 720, 1280, 90
    base = synth_frames_u8(6, H, W, seed=77)
    frames = [base[i % 6] for i in range(n)]
    got = {}
    tx, rx = S.loopback(_blob(), frames, H, W, 30.0, keep_symbols=True,
                        sink=lambda seq, fr: got.__setitem__(seq, fr))
    assert tx.frames_sent == n and rx.frames_received == n
    assert rx.frames_out_of_order == 0 and rx.gaps == 0 and rx.decode_failures == 0
    assert sorted(got) == list(range(n))
    for (seq, ys), ys_tx in zip(rx.y_symbols, tx.y_symbols):
        assert np.array_equal(ys, ys_tx)
    assert tx.late_frames == 0
    assert 29.0 <= tx.fps <= 31.0, tx.fps
    print(f"720p 1DN stream: {rx.fps:.1f} fps received, latency p50 {np.median(rx.latency_ms):.1f} ms, "
          f"{tx.bytes_sent / n / 1024:.1f} KiB/frame")


@pytest.mark.parametrize("kind", [1, 0])
def test_loopback_matches_direct_decode(S, kind):
    from paper_2208_01641_b200 import lic
    H, W, n = 200, 300, 12
    blob = _blob(kind=kind, act=0)
    frames = list(synth_frames_u8(n, H, W, seed=5))
    got = {}
    tx, rx = S.loopback(blob, frames, H, W, 200.0, keep_symbols=True, sink=lambda s, f: got.__setitem__(s, f))
    assert rx.frames_received == n and rx.gaps == 0 and rx.frames_out_of_order == 0
    c = lic.Codec(blob, H, W, max_batch=1)
    for i in range(n):
        out = np.empty((1, H, W, 3), np.uint8)
        c.decode(tx.y_symbols[i][None], out, u8=True)
        assert np.array_equal(out[0], got[i])
    c.close()


def test_digest_mismatch_aborts(S):
    import socket
    import threading
    H, W = 128, 128
    srv = socket.socket()
    srv.bind(("127.0.0.1", 0))
    srv.listen(1)
    port = srv.getsockname()[1]
    rx_coder = S.FrameCoder(_blob(seed=1), H, W)
    err = {}

    def rx():
        conn, _ = srv.accept()
        try:
            S.run_receiver(rx_coder, conn)
        except S.WireError as e:
            err["e"] = str(e)
        conn.close()

    th = threading.Thread(target=rx)
    th.start()
    tx_coder = S.FrameCoder(_blob(seed=2), H, W)
    cli = socket.create_connection(("127.0.0.1", port))
    try:
        S.run_sender(tx_coder, list(synth_frames_u8(2, H, W, seed=1)), cli, 100.0)
    except OSError:
        pass                                   # receiver may close first
    cli.close()
    th.join()
    srv.close()
    assert "digest" in err.get("e", "")


def test_corrupted_frame_is_counted(S):
    H, W, n = 128, 192, 8
    tx, rx = S.loopback(_blob(), list(synth_frames_u8(n, H, W, seed=9)), H, W, 200.0, corrupt_seq=3)
    assert rx.decode_failures == 1 and rx.frames_received == n - 1 and rx.gaps == 0


def test_received_stream_decodes_with_the_oracle(S):
    """PAPER.md:187-189 end to end against the oracle: the paper's demo codec (factorized +
    1DN, 1280x720) streamed at 30 FPS; one received frame's wire payload is decoded by the
    ORACLE (its rANS decoder over the 4 channel-slab substreams, R21, then g_s with
    1DN) and equals the receiver's frame (u8 +-1); the sender's symbols of that frame are the
    oracle encoder's (c18 tie rule)."""
    from oracle import oracle as O
    from parity import check_symbols
    from lic_synth import u8_to_f32_chw
    H, W, n, pick = 720, 1280, 6, 2
    spec = ModelSpec(kind=0, N=128, M=192, activation=ACT_1DN)
    w = generate_weights(spec, 0)
    frames = list(synth_frames_u8(n, H, W, seed=78))
    got = {}
    tx, rx = S.loopback(write_licw(spec, w), frames, H, W, 30.0, keep_symbols=True, keep_payloads=(pick,),
                        sink=lambda s, f: got.__setitem__(s, f))
    assert rx.frames_received == n and rx.gaps == 0 and rx.frames_out_of_order == 0
    k, ystr, zstr = S.unpack_frame(rx.payloads[pick])
    assert zstr is None
    tabs = O.build_tables(w, False, 32)
    xp, crop = O.pad_chw(u8_to_f32_chw(frames[pick][None])[0], hyper=False)
    y_shape = (192, xp.shape[1] // 16, xp.shape[2] // 16)
    xhat, ys = O.decode_strings(ystr, None, w, tabs, False, y_shape, None, crop, H, W, substreams=k, act=1)
    assert np.array_equal(ys, tx.y_symbols[pick])
    ref8 = np.floor(np.moveaxis(xhat, 0, -1).astype(np.float64) * 255 + 0.5)
    assert np.max(np.abs(got[pick].astype(np.int32) - ref8)) <= 1
    p = O.encode_planes(xp, w, False, 32, act=1)
    n_flip = check_symbols(tx.y_symbols[pick], p["y_sym"], p["y"] - w["mu_y"][:, None, None], what="stream y_sym")
    print(f"oracle decode of received frame {pick}: {len(ystr)} bytes, K = {k}, symbol flips vs oracle encode {n_flip}")
