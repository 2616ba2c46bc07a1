"""Multi-process host logic on CPU (gloo, world_size 2) -- -m "not gpu".

Frames shard by rank (t mod G) with no data-path collective; the end-of-run gather orders
the strings by frame index so the ordered set (and its digest) is the same for G = 1, 2.
The per-frame strings here are produced by the product host coder from seeded planes, so
the test exercises the real coder + gather path without a GPU.
"""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2208_01641_b200.dist import frames_for_rank, gather_bitstreams, stream_digest, verify_frames

N_FRAMES = 7


def _frame_strings(t):
    from paper_2208_01641_b200 import build
    build.build()
    from paper_2208_01641_b200 import lic
    from lic_synth import scale_table
    rng = np.random.default_rng(100 + t)
    cdf = lic.cdf_build(scale_table(), 32)
    idx = rng.integers(0, 20, 4096).astype(np.uint8)
    sym = np.clip(np.round(rng.standard_normal(4096) * scale_table()[idx]), -32, 32).astype(np.int8)
    y = lic.rans_encode(sym, cdf, rows=idx)
    zc = lic.cdf_build(np.full(8, 1.0, np.float32), 32)
    z = lic.rans_encode(np.clip(np.round(rng.standard_normal((8, 2, 2))), -32, 32).astype(np.int8), zc)
    return y, z


def _worker(rank, world, port, q, bench_path=False):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    if bench_path:
        # bench.py's end-of-run gather: local frame i of rank r is global frame r + G*i, the
        # verification run covers global frames 0..7 whoever holds them (batch 4)
        nv, keep = verify_frames(rank, world, 4, 8)
        assert nv % 4 == 0 and all(t < 8 for _, t in keep)
        local = {t: _frame_strings(t) for _, t in keep}
    else:
        local = {t: _frame_strings(t) for t in frames_for_rank(N_FRAMES, rank, world)}
    merged = gather_bitstreams(local, rank, world)
    if rank == 0:
        q.put(([i for i, _, _ in merged], stream_digest(merged)))
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_frames_for_rank_partition():
    for world in (1, 2, 3, 8):
        owned = sorted(t for r in range(world) for t in frames_for_rank(100, r, world))
        assert owned == list(range(100))
    with pytest.raises(ValueError):
        frames_for_rank(10, 2, 2)


def test_gather_world2_matches_world1():
    ref = gather_bitstreams({t: _frame_strings(t) for t in range(N_FRAMES)}, 0, 1)
    ref_digest = stream_digest(ref)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    idx, digest = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert idx == list(range(N_FRAMES))
    assert digest == ref_digest


def test_verify_frames_cover_the_same_set_for_every_world():
    """bench.py's gather set (global frames 0..7) is the same for G = 1, 2, 4, 8, so the
    gathered digest is G-invariant."""
    ref = stream_digest(gather_bitstreams({t: _frame_strings(t) for t in range(8)}, 0, 1))
    for world in (1, 2, 4, 8):
        merged = {}
        for r in range(world):
            nv, keep = verify_frames(r, world, 4, 8)
            assert nv >= 4 and nv % 4 == 0 and len(keep) <= nv
            for i, t in keep:
                assert t == r + world * i and t not in merged
                merged[t] = _frame_strings(t)
        assert sorted(merged) == list(range(8))
        assert stream_digest(gather_bitstreams(merged, 0, 1)) == ref


def test_bench_gather_world2_matches_world1():
    """The same path with two gloo processes (the NCCL path of bench.py uses the same calls)."""
    ref = stream_digest(gather_bitstreams({t: _frame_strings(t) for t in range(8)}, 0, 1))
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q, True)) for r in range(2)]
    for p in procs:
        p.start()
    idx, digest = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert idx == list(range(8))
    assert digest == ref
