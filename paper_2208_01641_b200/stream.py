"""Streaming demonstration (§VI, Fig. 4).

"We simulate a video monitoring system ... The devices transfer streams of video encoded by
learned image compression to a central server over TCP/IP networking.  The capturing side ...
encoding a 1280x720 stream at 30 FPS.  The stream is encoded by the factorized-prior model
with 1DN activation ... we encode every frame as keyframes"; "no frame drops
or noticeable jittering".

A sender paces synthetic frames at a target rate, encodes each through the C ABI (lic_encode_u8
on the GPU, then the native host rANS coder) and writes LICS messages on a TCP connection; a
receiver reads them, decodes (host rANS -> lic_hyper_indexes -> host rANS -> lic_decode_u8)
and hands frames to a sink in sequence order, counting gaps, reordering and decode failures.
This module is orchestration and framing only: every transform and coder step runs in
liblic.so.

Wire format (SPEC.md "stream" module, frozen at version 1; all integers little-endian):
  message   = "LICS" | version u8 = 1 | msg_type u8 (0 handshake, 1 frame, 2 end-of-stream)
              | sequence u64 | capture_timestamp_us u64 | payload_len u32 | payload
  handshake = codec_kind u8 | activation u8 | N u16 | M u16 | height u16 | width u16
              | target_fps u16 | weights_digest 32 B (SHA-256 of the LICW weights file)
  frame     = substreams u8 | y_len u32 | y string | z_len u32 | z string (z_len 0: factorized)
The y string is the lic_rans_encode_slabs framing with `substreams` channel slabs
(R21); z is one lic_rans_encode string.
"""
from __future__ import annotations

import hashlib
import socket
import struct
import threading
import time
from dataclasses import dataclass, field

import numpy as np

from . import lic

MAGIC = b"LICS"
VERSION = 1
MSG_HANDSHAKE, MSG_FRAME, MSG_END = 0, 1, 2
MAX_PAYLOAD = 64 << 20
_HDR = struct.Struct("<4sBBQQI")          # 26 bytes
_HS = struct.Struct("<BBHHHHH32s")        # 44 bytes


class WireError(Exception):
    pass


@dataclass
class Message:
    msg_type: int
    sequence: int
    timestamp_us: int
    payload: bytes = b""


def pack_message(m: Message) -> bytes:
    if len(m.payload) > MAX_PAYLOAD:
        raise WireError(f"payload {len(m.payload)} > {MAX_PAYLOAD}")
    return _HDR.pack(MAGIC, VERSION, m.msg_type, m.sequence, m.timestamp_us, len(m.payload)) + m.payload


def _recv_exact(sock, n, what):
    buf = bytearray()
    while len(buf) < n:
        chunk = sock.recv(n - len(buf))
        if not chunk:
            raise WireError(f"truncated {what}: expected {n} bytes, got {len(buf)}")
        buf += chunk
    return bytes(buf)


def read_message(sock) -> Message | None:
    """One message; None on a clean close before the first header byte."""
    first = sock.recv(1)
    if not first:
        return None
    head = first + _recv_exact(sock, _HDR.size - 1, "header")
    magic, ver, mtype, seq, ts, plen = _HDR.unpack(head)
    if magic != MAGIC:
        raise WireError(f"bad magic {magic!r}")
    if ver != VERSION:
        raise WireError(f"unsupported version {ver}")
    if plen > MAX_PAYLOAD:
        raise WireError(f"payload_len {plen} > {MAX_PAYLOAD}")
    return Message(mtype, seq, ts, _recv_exact(sock, plen, "payload"))


@dataclass
class Handshake:
    codec_kind: int
    activation: int
    N: int
    M: int
    height: int
    width: int
    target_fps: int
    digest: bytes

    def pack(self) -> bytes:
        return _HS.pack(self.codec_kind, self.activation, self.N, self.M, self.height, self.width,
                        self.target_fps, self.digest)

    @staticmethod
    def unpack(b: bytes) -> "Handshake":
        if len(b) != _HS.size:
            raise WireError(f"handshake of {len(b)} bytes")
        return Handshake(*_HS.unpack(b))


def weights_digest(licw: bytes) -> bytes:
    return hashlib.sha256(licw).digest()


def licw_header(licw: bytes):
    """(kind, activation, N, M) from the LICW header."""
    _, kind, act, N, M, _ = struct.unpack_from("<BBBHHH", licw, 4)
    return kind, act, N, M


def pack_frame(ystr: bytes, zstr: bytes | None, substreams: int) -> bytes:
    z = zstr or b""
    return struct.pack("<BI", substreams, len(ystr)) + ystr + struct.pack("<I", len(z)) + z


def unpack_frame(b: bytes):
    if len(b) < 9:
        raise WireError("frame payload too short")
    k, yl = struct.unpack_from("<BI", b, 0)
    if 5 + yl + 4 > len(b):
        raise WireError("frame payload: y string truncated")
    y = b[5:5 + yl]
    (zl,) = struct.unpack_from("<I", b, 5 + yl)
    if 9 + yl + zl != len(b):
        raise WireError("frame payload: bad z length")
    z = b[9 + yl:]
    return k, y, (z if zl else None)


# ---------------------------------------------------------------- codec sessions
class FrameCoder:
    """Per-frame encode / decode through the C ABI (batch 1): GPU transforms + host rANS."""

    def __init__(self, licw: bytes, height: int, width: int, device: int = 0, substreams: int = 4):
        self.licw = licw
        self.codec = lic.Codec(licw, height, width, max_batch=1, device=device)
        self.height, self.width = height, width
        self.hyper = self.codec.hyper
        self.substreams = substreams
        self.tab_y = lic.RansTables(self.codec.cdf(2 if self.hyper else 0))
        self.tab_z = lic.RansTables(self.codec.cdf(1)) if self.hyper else None
        self.ys = np.empty((1,) + self.codec.y_shape, np.int8)
        self.yi = np.empty((1,) + self.codec.y_shape, np.uint8) if self.hyper else None
        self.zs = np.empty((1,) + self.codec.z_shape, np.int8) if self.hyper else None
        self.out = np.empty((1, height, width, 3), np.uint8)

    def encode(self, frame_hwc_u8: np.ndarray):
        """-> (y string, z string | None, y symbols)"""
        self.codec.encode(np.ascontiguousarray(frame_hwc_u8[None]), self.ys, self.yi, self.zs, u8=True)
        y = self.tab_y.encode(self.ys[0], rows=None if not self.hyper else self.yi[0], substreams=self.substreams)
        z = self.tab_z.encode(self.zs[0]) if self.hyper else None
        return y, z, self.ys[0].copy()

    def decode(self, ystr: bytes, zstr: bytes | None, substreams: int):
        """-> (frame u8 HWC, y symbols); raises lic.CorruptStream / WireError on bad strings."""
        if self.hyper:
            if zstr is None:
                raise WireError("hyperprior frame without a z string")
            zs = self.tab_z.decode(zstr, self.codec.z_shape)
            idx = np.empty((1,) + self.codec.y_shape, np.uint8)
            self.codec.hyper_indexes(zs[None], idx)
            ys = self.tab_y.decode(ystr, self.codec.y_shape, rows=idx[0], substreams=substreams)
        else:
            ys = self.tab_y.decode(ystr, self.codec.y_shape, substreams=substreams)
        self.codec.decode(ys[None], self.out, u8=True)
        return self.out[0].copy(), ys

    def close(self):
        self.codec.close()


@dataclass
class SenderStats:
    frames_sent: int = 0
    late_frames: int = 0
    seconds: float = 0.0
    bytes_sent: int = 0
    y_symbols: list = field(default_factory=list)      # per frame, when keep_symbols

    @property
    def fps(self):
        return self.frames_sent / self.seconds if self.seconds else 0.0


@dataclass
class ReceiverStats:
    frames_received: int = 0
    frames_out_of_order: int = 0
    gaps: int = 0
    decode_failures: int = 0
    seconds: float = 0.0
    latency_ms: list = field(default_factory=list)
    handshake: Handshake | None = None
    y_symbols: list = field(default_factory=list)
    payloads: dict = field(default_factory=dict)        # sequence -> frame payload (keep_payloads)

    @property
    def fps(self):
        return self.frames_received / self.seconds if self.seconds else 0.0


def _now_us():
    return time.monotonic_ns() // 1000


def run_sender(coder: FrameCoder, frames, sock, target_fps: float, keep_symbols=False, corrupt_seq=None):
    """PAPER.md:187 capture side: pace `frames` (iterable of u8 HxWx3) at target_fps on a
    monotonic clock, encode each, send LICS messages in order, then end-of-stream.  A frame
    whose encode finishes after its next frame's slot is counted late, never dropped.
    corrupt_seq: test-only fault injection (flip bytes in that frame's y string)."""
    st = SenderStats()
    kind, act, N, M = licw_header(coder.licw)
    hs = Handshake(kind, act, N, M, coder.height, coder.width, int(round(target_fps)), weights_digest(coder.licw))
    sock.sendall(pack_message(Message(MSG_HANDSHAKE, 0, _now_us(), hs.pack())))
    period = 1.0 / target_fps
    t0 = time.monotonic()
    seq = 0
    for fr in frames:
        slot = t0 + seq * period
        now = time.monotonic()
        if now < slot:
            time.sleep(slot - now)
        cap = _now_us()
        y, z, ys = coder.encode(fr)
        if corrupt_seq is not None and seq == corrupt_seq:
            yb = bytearray(y)
            for i in range(8, min(len(yb), 64)):
                yb[i] ^= 0x5A
            y = bytes(yb)
        msg = pack_message(Message(MSG_FRAME, seq, cap, pack_frame(y, z, coder.substreams)))
        sock.sendall(msg)
        st.bytes_sent += len(msg)
        if keep_symbols:
            st.y_symbols.append(ys)
        if time.monotonic() > slot + period:
            st.late_frames += 1
        seq += 1
    sock.sendall(pack_message(Message(MSG_END, seq, _now_us(), b"")))
    st.frames_sent = seq
    st.seconds = time.monotonic() - t0
    return st


def run_receiver(coder: FrameCoder, sock, sink=None, keep_symbols=False, keep_payloads=()):
    """PAPER.md:187 server side: validate the handshake against the local weights, decode every
    frame message, deliver (sequence, frame) to `sink` in order; gaps and reordering are
    counted, a frame that fails to decode is counted and skipped (the stream continues)."""
    st = ReceiverStats()
    m = read_message(sock)
    if m is None or m.msg_type != MSG_HANDSHAKE:
        raise WireError("stream does not start with a handshake")
    hs = Handshake.unpack(m.payload)
    st.handshake = hs
    if hs.digest != weights_digest(coder.licw):
        raise WireError("weights digest mismatch")
    if (hs.height, hs.width) != (coder.height, coder.width):
        raise WireError(f"geometry {hs.height}x{hs.width} != {coder.height}x{coder.width}")
    expect = 0
    t0 = None
    while True:
        m = read_message(sock)
        if m is None or m.msg_type == MSG_END:
            break
        if m.msg_type != MSG_FRAME:
            raise WireError(f"unexpected message type {m.msg_type}")
        if t0 is None:
            t0 = time.monotonic()
        if m.sequence != expect:
            if m.sequence < expect:
                st.frames_out_of_order += 1
            else:
                st.gaps += m.sequence - expect
        expect = max(expect, m.sequence + 1)
        if m.sequence in keep_payloads:
            st.payloads[m.sequence] = m.payload
        try:
            k, y, z = unpack_frame(m.payload)
            frame, ys = coder.decode(y, z, k)
        except (lic.CorruptStream, lic.LicError, WireError):
            st.decode_failures += 1
            continue
        st.frames_received += 1
        st.latency_ms.append((_now_us() - m.timestamp_us) / 1e3)     # loopback: one monotonic clock
        if keep_symbols:
            st.y_symbols.append((m.sequence, ys))
        if sink is not None:
            sink(m.sequence, frame)
    st.seconds = (time.monotonic() - t0) if t0 is not None else 0.0
    return st


def loopback(licw: bytes, frames, height: int, width: int, target_fps: float, device: int = 0,
             substreams: int = 4, keep_symbols=False, corrupt_seq=None, sink=None, keep_payloads=()):
    """Sender and receiver on 127.0.0.1 in one process (two threads, one codec each)."""
    srv = socket.socket(socket.AF_INET, socket.SOCK_STREAM)
    srv.bind(("127.0.0.1", 0))
    srv.listen(1)
    port = srv.getsockname()[1]
    rx_coder = FrameCoder(licw, height, width, device, substreams)
    result = {}

    def rx():
        conn, _ = srv.accept()
        try:
            result["rx"] = run_receiver(rx_coder, conn, sink=sink, keep_symbols=keep_symbols,
                                        keep_payloads=keep_payloads)
        except Exception as e:          # surfaced to the caller below
            result["rx_err"] = e
        finally:
            conn.close()

    th = threading.Thread(target=rx)
    th.start()
    tx_coder = FrameCoder(licw, height, width, device, substreams)
    cli = socket.create_connection(("127.0.0.1", port))
    cli.setsockopt(socket.IPPROTO_TCP, socket.TCP_NODELAY, 1)
    try:
        tx = run_sender(tx_coder, frames, cli, target_fps, keep_symbols=keep_symbols, corrupt_seq=corrupt_seq)
    finally:
        cli.close()
    th.join()
    srv.close()
    tx_coder.close()
    rx_coder.close()
    if "rx_err" in result:
        raise result["rx_err"]
    return tx, result["rx"]
