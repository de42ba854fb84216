"""Utterance sharder (paper_1702_07825_b200/shard.py): block partition properties and
the gather path on a real 2-process gloo group (CPU), the multi-GPU plumbing without
GPUs.  Generation itself is per-utterance independent, which the GPU
tests pin bitwise (test_gpu_parity.py position-independence tests)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1702_07825_b200.shard import gather_codes, shard_range


@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
@pytest.mark.parametrize("n", [0, 1, 5, 8, 255, 2048])
def test_shard_range_partitions(n, world):
    blocks = [shard_range(n, world, r) for r in range(world)]
    pos = 0
    for start, count in blocks:
        assert start == pos and count >= 0
        pos += count
    assert pos == n
    sizes = [c for _, c in blocks]
    assert max(sizes) - min(sizes) <= 1
    assert sizes == sorted(sizes, reverse=True)


def test_shard_range_rejects_bad_args():
    with pytest.raises(ValueError):
        shard_range(4, 0, 0)
    with pytest.raises(ValueError):
        shard_range(4, 2, 2)
    with pytest.raises(ValueError):
        shard_range(-1, 2, 0)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n_utts, N, q):
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        start, count = shard_range(n_utts, world, rank)
        # stand-in for this shard's generated codes: row u holds (u * 7 + n) mod 256
        local = torch.tensor([[(u * 7 + n) % 256 for n in range(N)] for u in range(start, start + count)],
                             dtype=torch.uint8).reshape(count, N)
        full = gather_codes(local, n_utts)
        if rank == 0:
            q.put(full.numpy().tolist())
        else:
            q.put(None if full is None else "non-root got data")
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n_utts", [2, 5, 1])
def test_gather_codes_gloo_world2(n_utts):
    world, N = 2, 9
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n_utts, N, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    rows = [g for g in got if g is not None]
    assert len(rows) == 1, got
    expect = np.array([[(u * 7 + n) % 256 for n in range(N)] for u in range(n_utts)], np.uint8)
    assert np.array_equal(np.array(rows[0], np.uint8), expect)


def test_gather_codes_single_process_is_identity():
    local = torch.arange(12, dtype=torch.uint8).reshape(3, 4)
    assert gather_codes(local, 3) is local
