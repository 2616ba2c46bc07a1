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
