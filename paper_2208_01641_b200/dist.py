"""Multi-GPU host logic: frame sharding and the end-of-run bitstream gather.

The path shards by frame (every frame is a keyframe): with G processes (one
per GPU, torchrun), frame t belongs to rank t mod G; there is no collective on the data
path.  At the end of a run the per-frame strings (or their digests) are gathered to rank
0 and ordered by frame index; the ordered set is independent of G.
"""
from __future__ import annotations

import hashlib


def frames_for_rank(n_total: int, rank: int, world: int) -> list[int]:
    """Global frame indices owned by `rank` (t = rank, rank + G, ...)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    return list(range(rank, n_total, world))


def gather_bitstreams(local: dict, rank: int, world: int, group=None):
    """local: {frame index: (y_bytes, z_bytes or None)}.  Returns, on rank 0, the list of
    (index, y, z) over all ranks ordered by index (None elsewhere).  Uses
    torch.distributed.gather_object (NCCL over NVLink or gloo)."""
    items = sorted(local.items())
    if world == 1:
        return [(i, y, z) for i, (y, z) in items]
    import torch.distributed as dist
    out = [None] * world if rank == 0 else None
    dist.gather_object(items, out, dst=0, group=group)
    if rank != 0:
        return None
    merged = [(i, y, z) for part in out for i, (y, z) in part]
    merged.sort(key=lambda r: r[0])
    idx = [i for i, _, _ in merged]
    if len(set(idx)) != len(idx):
        raise RuntimeError("duplicate frame index in gather")
    return merged


def stream_digest(ordered) -> str:
    """sha256 over (index, len(y), y, len(z), z) in index order: equal for every G."""
    h = hashlib.sha256()
    for i, y, z in ordered:
        z = z or b""
        h.update(i.to_bytes(8, "little"))
        h.update(len(y).to_bytes(8, "little"))
        h.update(y)
        h.update(len(z).to_bytes(8, "little"))
        h.update(z)
    return h.hexdigest()


def verify_frames(rank: int, world: int, batch: int, n_global: int):
    """Frames of the end-of-run bitstream gather: global frames 0 .. n_global-1 whoever holds
    them, so the gathered, ordered set is the same for every G.  Rank r's local frame i is
    global frame t = r + G * i; it runs `nv` local frames (whole batches, at least one) and
    keeps [(i, t)] for t < n_global.  Returns (nv, keep)."""
    if world < 1 or not 0 <= rank < world or batch < 1:
        raise ValueError("bad rank/world/batch")
    keep = [(i, rank + world * i) for i in range(n_global) if rank + world * i < n_global]
    nv = max(batch, -(-len(keep) // batch) * batch)
    return nv, keep
