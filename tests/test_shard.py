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


# ---- counter-based batched inputs (synth.make_batch_hashed_torch): keyed per (role, utterance)
def test_hashed_inputs_host_equals_device_recipe_and_independent_of_batch():
    from paper_1702_07825_b200 import synth
    cfg = synth.Config(3, 8, 16)
    N, hop = 200, 16
    full_c, full_u = synth.make_batch_hashed_torch(cfg, N, list(range(10)), hop, "cpu")
    # the same utterances in another batch composition / order / shard: identical values
    sub_c, sub_u = synth.make_batch_hashed_torch(cfg, N, [7, 2, 9], hop, "cpu")
    for i, u in enumerate([7, 2, 9]):
        assert torch.equal(sub_c[i], full_c[u]) and torch.equal(sub_u[i], full_u[u])
        # host recipe equals the torch (device) recipe element for element
        np.testing.assert_array_equal(synth.make_cond_hashed(cfg, synth.n_frames_for(N, hop), u), sub_c[i].numpy())
        np.testing.assert_array_equal(synth.make_uniforms_hashed(N, u), sub_u[i].numpy())
    # ranges: cond in [-0.5, 0.5), uniforms in [0, 1) on the 2^-24 grid; utterances differ
    assert float(full_c.min()) >= -0.5 and float(full_c.max()) < 0.5
    assert float(full_u.min()) >= 0.0 and float(full_u.max()) < 1.0
    assert torch.all(full_u * 2 ** 24 == torch.floor(full_u * 2 ** 24))
    assert not torch.equal(full_u[0], full_u[1]) and not torch.equal(full_c[0], full_c[1])


def test_hashed_uniforms_look_uniform():
    from paper_1702_07825_b200 import synth
    x = synth.make_uniforms_hashed(1 << 18, 11).astype(np.float64)
    assert abs(x.mean() - 0.5) < 0.003 and abs(x.var() - 1 / 12) < 0.002
    hist = np.bincount((x * 64).astype(int), minlength=64)
    assert np.all(np.abs(hist - x.size / 64) < 6 * np.sqrt(x.size / 64))
    assert abs(np.corrcoef(x[:-1], x[1:])[0, 1]) < 0.01
    # the role and utterance keys decorrelate streams
    y = synth.make_uniforms_hashed(1 << 18, 12).astype(np.float64)
    assert abs(np.corrcoef(x, y)[0, 1]) < 0.01


def test_generate_sharded_simulated_ranks_cover_the_utterances():
    """generate_sharded with an explicit (world, rank) runs exactly that shard's utterances."""
    from paper_1702_07825_b200.shard import generate_sharded

    class Fake:
        def generate(self, cond, u, hop):
            return (cond[:, 0, 0, :u.shape[1]] * 0 + torch.tensor([float(x) for x in seen[-1]])[:, None]).to(torch.uint8)

    seen = []

    def make_inputs(ids):
        seen.append(list(ids))
        return torch.zeros((len(ids), 1, 1, 4)), torch.zeros((len(ids), 4))

    rows = []
    for k in range(3):
        local, full, (start, count) = generate_sharded(Fake(), make_inputs, 10, 4, 1, world=3, rank=k)
        assert full is None and local.shape == (count, 4)
        rows += local[:, 0].tolist()
    assert rows == list(range(10))
