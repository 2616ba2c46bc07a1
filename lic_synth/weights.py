"""Random-init model parameters and the LICW weight container.

Container ("Weight file: magic LICW; version u8 = 1; codec_kind u8;
activation u8; N u16; M u16; L u16; then each parameter block as (tag u8,
element-count u32, raw 32-bit little-endian floats) in a fixed documented
order").  The fixed order is ``BLOCKS`` below; factorized files omit the
hyper-only blocks.  Everything is little-endian.

Architecture: CompressAI bmshj2018 shapes
  g_a : conv5x5/s2 3->N, GDN, conv N->N, GDN, conv N->N, GDN, conv N->M
  g_s : deconv5x5/s2 M->N, IGDN, deconv N->N, IGDN, deconv N->N, IGDN, deconv N->3
  h_a : conv3x3/s1 M->N, ReLU, conv5x5/s2 N->N, ReLU, conv5x5/s2 N->N   (input |y|)
  h_s : deconv5x5/s2 N->N, ReLU, deconv N->N, ReLU, conv3x3/s1 N->M, ReLU
All conv and deconv weights are stored out x in x k x k.

Initialisation: SURVEY.md §8(c) reading c15 (SPEC.md:305's a = sqrt(1/fan_in) is
degenerate: every symbol quantises to 0).  The north star asks for "weights
randomly initialised with positive GDN beta/gamma".  Conv/deconv weights are
rounded to fp16-representable values (exact fp16 B operands on the GPU; the
oracle reads the same fp32 numbers).
"""
from __future__ import annotations

import hashlib
import struct
from dataclasses import dataclass

import numpy as np

MAGIC = b"LICW"
VERSION = 1
KIND_FACTORIZED = 0
KIND_HYPER = 1
ACT_GDN = 0
ACT_1DN = 1
N_SCALES = 64
SCALE_MIN = 0.11
SCALE_MAX = 256.0


@dataclass(frozen=True)
class ModelSpec:
    kind: int          # 0 factorized, 1 hyperprior
    N: int
    M: int
    L: int = 32        # symbol support [-L, L]
    activation: int = ACT_GDN


# (tag, name, shape-fn(N, M), hyper_only, kind)
#   kind: "conv"/"deconv" weight (with k, stride), "bias", "beta", "gamma", "param"
def _blocks():
    b = []
    t = [0]

    def add(name, shape, hyper_only, role, k=0, stride=0):
        t[0] += 1
        b.append(dict(tag=t[0], name=name, shape=shape, hyper_only=hyper_only, role=role,
                      k=k, stride=stride))

    # g_a
    add("ga1.w", lambda N, M: (N, 3, 5, 5), False, "conv", 5, 2)
    add("ga1.b", lambda N, M: (N,), False, "bias")
    add("ga1.beta", lambda N, M: (N,), False, "beta")
    add("ga1.gamma", lambda N, M: (N, N), False, "gamma")
    add("ga2.w", lambda N, M: (N, N, 5, 5), False, "conv", 5, 2)
    add("ga2.b", lambda N, M: (N,), False, "bias")
    add("ga2.beta", lambda N, M: (N,), False, "beta")
    add("ga2.gamma", lambda N, M: (N, N), False, "gamma")
    add("ga3.w", lambda N, M: (N, N, 5, 5), False, "conv", 5, 2)
    add("ga3.b", lambda N, M: (N,), False, "bias")
    add("ga3.beta", lambda N, M: (N,), False, "beta")
    add("ga3.gamma", lambda N, M: (N, N), False, "gamma")
    add("ga4.w", lambda N, M: (M, N, 5, 5), False, "conv", 5, 2)
    add("ga4.b", lambda N, M: (M,), False, "bias")
    # g_s
    add("gs1.w", lambda N, M: (N, M, 5, 5), False, "deconv", 5, 2)
    add("gs1.b", lambda N, M: (N,), False, "bias")
    add("gs1.beta", lambda N, M: (N,), False, "beta")
    add("gs1.gamma", lambda N, M: (N, N), False, "gamma")
    add("gs2.w", lambda N, M: (N, N, 5, 5), False, "deconv", 5, 2)
    add("gs2.b", lambda N, M: (N,), False, "bias")
    add("gs2.beta", lambda N, M: (N,), False, "beta")
    add("gs2.gamma", lambda N, M: (N, N), False, "gamma")
    add("gs3.w", lambda N, M: (N, N, 5, 5), False, "deconv", 5, 2)
    add("gs3.b", lambda N, M: (N,), False, "bias")
    add("gs3.beta", lambda N, M: (N,), False, "beta")
    add("gs3.gamma", lambda N, M: (N, N), False, "gamma")
    add("gs4.w", lambda N, M: (3, N, 5, 5), False, "deconv", 5, 2)
    add("gs4.b", lambda N, M: (3,), False, "bias")
    # h_a
    add("ha1.w", lambda N, M: (N, M, 3, 3), True, "conv", 3, 1)
    add("ha1.b", lambda N, M: (N,), True, "bias")
    add("ha2.w", lambda N, M: (N, N, 5, 5), True, "conv", 5, 2)
    add("ha2.b", lambda N, M: (N,), True, "bias")
    add("ha3.w", lambda N, M: (N, N, 5, 5), True, "conv", 5, 2)
    add("ha3.b", lambda N, M: (N,), True, "bias")
    # h_s
    add("hs1.w", lambda N, M: (N, N, 5, 5), True, "deconv", 5, 2)
    add("hs1.b", lambda N, M: (N,), True, "bias")
    add("hs2.w", lambda N, M: (N, N, 5, 5), True, "deconv", 5, 2)
    add("hs2.b", lambda N, M: (N,), True, "bias")
    add("hs3.w", lambda N, M: (M, N, 3, 3), True, "conv", 3, 1)
    add("hs3.b", lambda N, M: (M,), True, "bias")
    # entropy-model parameters
    add("mu_y", lambda N, M: (M,), False, "param")       # fact: mu_c; hyper: zeros
    add("sigma_y", lambda N, M: (M,), False, "param")    # fact: sigma_c; hyper: ones (unused)
    add("mu_z", lambda N, M: (N,), True, "param")
    add("sigma_z", lambda N, M: (N,), True, "param")
    add("scale_table", lambda N, M: (N_SCALES,), False, "param")
    return b


BLOCKS = _blocks()


def block_specs(spec: ModelSpec):
    """The ordered list of (tag, name, shape) present in a file of this spec."""
    out = []
    for b in BLOCKS:
        if b["hyper_only"] and spec.kind != KIND_HYPER:
            continue
        out.append((b["tag"], b["name"], tuple(b["shape"](spec.N, spec.M))))
    return out


def scale_table() -> np.ndarray:
    """64 log-spaced scales in [0.11, 256]:
    fp32(exp(ln 0.11 + i*(ln 256 - ln 0.11)/63)), computed in fp64."""
    lo, hi = np.log(SCALE_MIN), np.log(SCALE_MAX)
    i = np.arange(N_SCALES, dtype=np.float64)
    return np.exp(lo + i * (hi - lo) / (N_SCALES - 1)).astype(np.float32)


def _fp16_exact(a: np.ndarray) -> np.ndarray:
    return a.astype(np.float16).astype(np.float32)


def generate_weights(spec: ModelSpec, seed: int = 0) -> dict:
    """Random-init weights per SURVEY.md §8(c) reading c15 (numpy PCG64, seeded).

    conv/deconv W ~ U[-a, a], a = sqrt(3 / fan_in_eff), fan_in_eff = Cin*k^2 (conv)
    or Cin*k^2/4 (stride-2 deconv), rounded to fp16-representable; bias fp32 U[-a, a].
    GDN/IGDN: beta_i = 1 + 0.1*U[0,1); gamma = 0.1*I + (0.1/C)*U[0,1) (fp16-exact).
    h_s L3 bias += 1.0; g_s L4 weights x0.25 and bias 0.5.
    sigma_c, sigma_z ~ U[0.5, 1.5]; mu_c, mu_z ~ U[-0.25, 0.25] (hyper mu_y = 0).
    """
    rng = np.random.Generator(np.random.PCG64(seed))
    out = {}
    for tag, name, shape in block_specs(spec):
        b = next(x for x in BLOCKS if x["tag"] == tag)
        role = b["role"]
        if role in ("conv", "deconv"):
            cout, cin, k, _ = shape
            fan = cin * k * k if role == "conv" else cin * k * k / 4.0
            a = np.sqrt(3.0 / fan)
            w = rng.uniform(-a, a, size=shape)
            if name == "gs4.w":
                w = w * 0.25
            out[name] = _fp16_exact(w)
            out["__a_" + name[:-2]] = a
        elif role == "bias":
            layer = name[:-2]
            a = out["__a_" + layer]
            bb = rng.uniform(-a, a, size=shape).astype(np.float32)
            if name == "hs3.b":
                bb = bb + np.float32(1.0)
            if name == "gs4.b":
                bb = np.full(shape, 0.5, dtype=np.float32)
            out[name] = bb.astype(np.float32)
        elif role == "beta":
            out[name] = (1.0 + 0.1 * rng.uniform(0.0, 1.0, size=shape)).astype(np.float32)
        elif role == "gamma":
            C = shape[0]
            g = 0.1 * np.eye(C) + (0.1 / C) * rng.uniform(0.0, 1.0, size=shape)
            out[name] = _fp16_exact(g)
        else:
            if name == "scale_table":
                out[name] = scale_table()
            elif name == "mu_y":
                if spec.kind == KIND_HYPER:
                    out[name] = np.zeros(shape, np.float32)
                else:
                    out[name] = rng.uniform(-0.25, 0.25, size=shape).astype(np.float32)
            elif name == "sigma_y":
                if spec.kind == KIND_HYPER:
                    out[name] = np.ones(shape, np.float32)
                else:
                    out[name] = rng.uniform(0.5, 1.5, size=shape).astype(np.float32)
            elif name == "mu_z":
                out[name] = rng.uniform(-0.25, 0.25, size=shape).astype(np.float32)
            elif name == "sigma_z":
                out[name] = rng.uniform(0.5, 1.5, size=shape).astype(np.float32)
    for k in [k for k in out if k.startswith("__")]:
        del out[k]
    return out


def write_licw(spec: ModelSpec, weights: dict) -> bytes:
    """Serialise to the LICW container (little-endian)."""
    parts = [MAGIC, struct.pack("<BBBHHH", VERSION, spec.kind, spec.activation,
                                spec.N, spec.M, spec.L)]
    for tag, name, shape in block_specs(spec):
        a = np.ascontiguousarray(weights[name], dtype="<f4")
        assert a.shape == shape, (name, a.shape, shape)
        parts.append(struct.pack("<BI", tag, a.size))
        parts.append(a.tobytes())
    return b"".join(parts)


def read_licw_blocks(blob: bytes):
    """Parse an LICW blob into (ModelSpec, {name: array}).  Used by tests only."""
    if blob[:4] != MAGIC:
        raise ValueError("bad magic")
    ver, kind, act, N, M, L = struct.unpack_from("<BBBHHH", blob, 4)
    if ver != VERSION:
        raise ValueError("bad version")
    spec = ModelSpec(kind=kind, N=N, M=M, L=L, activation=act)
    off = 4 + 9
    out = {}
    for tag, name, shape in block_specs(spec):
        t, n = struct.unpack_from("<BI", blob, off)
        off += 5
        if t != tag or n != int(np.prod(shape)):
            raise ValueError(f"block {name}: tag {t} count {n}")
        out[name] = np.frombuffer(blob, dtype="<f4", count=n, offset=off).reshape(shape).copy()
        off += 4 * n
    if off != len(blob):
        raise ValueError("trailing bytes")
    return spec, out


def licw_digest(blob: bytes) -> bytes:
    """32-byte digest of the canonical file bytes."""
    return hashlib.sha256(blob).digest()
