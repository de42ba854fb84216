"""Utterance sharder: independent utterances across the GPUs of one box.

Generation of one utterance never needs another's data (each
utterance is its own auto-regressive process), so the batched path shards
*utterances*, one process per GPU, with no collective on the generation path
(BASELINE.json north_star: "Independent utterances shard across the 8 GPUs of one
box with no collective on the path and NCCL used only to gather results").

    start, count = shard_range(n_utts, world, rank)      # contiguous, balanced
    codes = generate_sharded(model, make_inputs, n_utts, N, hop)  # rank 0 gets all

`make_inputs(utt_ids)` returns (cond, uniforms) for those utterances (host or
device arrays); each rank builds only its own shard's inputs.  Gathering uses
torch.distributed (NCCL on GPUs, gloo on CPU) and happens after the timed work.
"""
from __future__ import annotations

from typing import Callable, Optional, Sequence, Tuple

import torch


def shard_range(n_utts: int, world: int, rank: int) -> Tuple[int, int]:
    """Contiguous block of utterances for `rank`: the first n_utts % world ranks
    take one extra, so block sizes differ by at most one and cover [0, n_utts)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of world {world}")
    if n_utts < 0:
        raise ValueError("n_utts must be >= 0")
    base, extra = divmod(n_utts, world)
    start = rank * base + min(rank, extra)
    return start, base + (1 if rank < extra else 0)


def _dist():
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized():
        return dist, dist.get_world_size(), dist.get_rank()
    return None, 1, 0


def gather_codes(local: torch.Tensor, n_utts: int, group=None) -> Optional[torch.Tensor]:
    """Reassemble per-rank code blocks [count, N] (uint8) into [n_utts, N] on rank 0
    (None elsewhere), in utterance order.  Blocks are padded to the largest shard
    for the all_gather and trimmed afterwards."""
    dist, world, rank = _dist()
    if dist is None:
        return local
    N = local.shape[1]
    biggest = shard_range(n_utts, world, 0)[1]
    pad = torch.zeros((biggest, N), dtype=local.dtype, device=local.device)
    pad[: local.shape[0]] = local
    parts = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(parts, pad, group=group)
    if rank != 0:
        return None
    out = [parts[r][: shard_range(n_utts, world, r)[1]] for r in range(world)]
    return torch.cat(out, 0)


def generate_sharded(model, make_inputs: Callable[[Sequence[int]], Tuple[torch.Tensor, torch.Tensor]],
                     n_utts: int, n_samples: int, hop: int, gather: bool = True, group=None,
                     world: Optional[int] = None, rank: Optional[int] = None):
    """Generate this rank's shard with one batched dvw_generate call; optionally
    gather all codes to rank 0.  Returns (local_codes, gathered_or_None, (start, count)).
    world / rank override the process group's (a single process simulating one shard of a
    G-GPU run, as the sharding-invariance test does); gathering needs the real group."""
    _, w0, r0 = _dist()
    world = w0 if world is None else world
    rank = r0 if rank is None else rank
    start, count = shard_range(n_utts, world, rank)
    if count == 0:
        local = torch.empty((0, n_samples), dtype=torch.uint8, device="cuda")
    else:
        cond, u = make_inputs(list(range(start, start + count)))
        local = model.generate(cond, u, hop)
    full = gather_codes(local, n_utts, group) if (gather and world == w0) else None
    return local, full, (start, count)
