"""LICS wire protocol of the streaming demonstration (§VI; SPEC.md "stream"
module) -- framing only, -m "not gpu"."""
import socket
import struct

import numpy as np
import pytest

from paper_2208_01641_b200 import stream as S


def _pair():
    a, b = socket.socketpair()
    return a, b


def test_message_roundtrip_and_magic():
    rng = np.random.default_rng(3)
    a, b = _pair()
    msgs = [S.Message(S.MSG_HANDSHAKE, 0, 17, b"\x01" * 44)]
    for i in range(20):
        msgs.append(S.Message(S.MSG_FRAME, i, int(rng.integers(0, 2 ** 62)), rng.bytes(int(rng.integers(0, 5000)))))
    msgs.append(S.Message(S.MSG_END, 20, 5, b""))
    wire = b"".join(S.pack_message(m) for m in msgs)
    assert wire[:4] == b"\x4c\x49\x43\x53"                       # "LICS"
    a.sendall(wire)
    a.close()
    got = []
    while True:
        m = S.read_message(b)
        if m is None:
            break
        got.append(m)
    assert got == msgs
    b.close()


def test_header_is_little_endian():
    w = S.pack_message(S.Message(S.MSG_FRAME, 0x0102030405060708, 9, b"xyz"))
    assert w[4] == 1 and w[5] == S.MSG_FRAME
    assert w[6:14] == bytes([8, 7, 6, 5, 4, 3, 2, 1])
    assert struct.unpack_from("<I", w, 22)[0] == 3 and w[26:] == b"xyz"


@pytest.mark.parametrize("bad,what", [
    (lambda w: b"LICX" + w[4:], "magic"),
    (lambda w: w[:4] + b"\x02" + w[5:], "version"),
    (lambda w: w[:-2], "truncated payload"),
    (lambda w: w[:10], "truncated header"),
    (lambda w: w[:22] + struct.pack("<I", (64 << 20) + 1) + w[26:], "payload_len"),
])
def test_read_errors(bad, what):
    a, b = _pair()
    a.sendall(bad(S.pack_message(S.Message(S.MSG_FRAME, 1, 2, b"hello world"))))
    a.close()
    with pytest.raises(S.WireError):
        S.read_message(b)
    b.close()


def test_payload_guard_on_write():
    with pytest.raises(S.WireError):
        S.pack_message(S.Message(S.MSG_FRAME, 0, 0, b"\0" * ((64 << 20) + 1)))


def test_handshake_and_frame_payloads():
    h = S.Handshake(0, 1, 128, 192, 720, 1280, 30, bytes(range(32)))
    assert S.Handshake.unpack(h.pack()) == h and len(h.pack()) == 44
    for z in (None, b"zz"):
        p = S.pack_frame(b"y" * 10, z, 4)
        assert S.unpack_frame(p) == (4, b"y" * 10, z)
    with pytest.raises(S.WireError):
        S.unpack_frame(S.pack_frame(b"y" * 10, b"zz", 4)[:-1])
