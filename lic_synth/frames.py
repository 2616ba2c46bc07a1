"""Synthetic u8 RGB frames (SURVEY.md §8(d) "Synthetic inputs").

Integer arithmetic, seed s, frame t, image H x W (HWC, u8):
  R = (x*255) // (W-1)
  G = (y*255) // (H-1)
  B = (((x + y + 4t) mod (H+W)) * 255) // (H+W)        (gradient moves with t)
plus uniform integer noise in [-12, 12] drawn from numpy PCG64 seeded with
[seed, t], then clamped to 0..255.  The paper loops a single sample image
("a 768x512 and a 1280x720 sample image as input in an infinite
loop"); streams use T frames looped.
"""
from __future__ import annotations

import numpy as np


def synth_frame_u8(H: int, W: int, seed: int = 0, t: int = 0) -> np.ndarray:
    y = np.arange(H, dtype=np.int64)[:, None]
    x = np.arange(W, dtype=np.int64)[None, :]
    r = (x * 255) // max(W - 1, 1) + 0 * y
    g = (y * 255) // max(H - 1, 1) + 0 * x
    b = (((x + y + 4 * t) % (H + W)) * 255) // (H + W)
    img = np.stack([r, g, b], axis=-1)
    rng = np.random.Generator(np.random.PCG64([seed, t]))
    img = img + rng.integers(-12, 13, size=img.shape)
    return np.clip(img, 0, 255).astype(np.uint8)


def synth_frames_u8(n: int, H: int, W: int, seed: int = 0, t0: int = 0) -> np.ndarray:
    """n frames, [n, H, W, 3] u8."""
    return np.stack([synth_frame_u8(H, W, seed, t0 + i) for i in range(n)])


def u8_to_f32_chw(frames_u8: np.ndarray) -> np.ndarray:
    """Float input frames for the f32 entry points: [n,H,W,3] u8 -> [n,3,H,W]
    fp32 in [0,1] (fp32(u8) / fp32(255), IEEE division)."""
    f = np.ascontiguousarray(np.moveaxis(frames_u8, -1, -3)).astype(np.float32)
    return f / np.float32(255.0)
