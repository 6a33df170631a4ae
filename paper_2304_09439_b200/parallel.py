"""Pair-batch sharding across ranks (one process per GPU) — SURVEY.md §8(e).

Pairs are independent, so a global batch of N pairs is split into contiguous shards of ceil(N/world)
pairs; each rank runs its shard through its own library context on its own GPU.  The path itself has
no collective.  `gather=True` reassembles the full result on every rank with one all_gather of
probs + labels (5 B/pair; NCCL over NVLink on GPUs, gloo in the CPU tests) — a convenience for callers
that need the whole answer on every rank.
"""
from __future__ import annotations

import numpy as np


def shard_bounds(N: int, world: int, rank: int):
    """[lo, hi) of rank's contiguous shard; shards have ceil(N/world) pairs, the last ones may be
    shorter or empty."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    per = -(-N // world) if N else 0
    lo = min(N, rank * per)
    return lo, min(N, lo + per)


def query_sharded(query_fn, pairs, poses, rank: int, world: int, gather: bool = True, group=None,
                  device=None):
    """Run `query_fn(pairs_shard, poses_shard) -> (probs float32, labels uint8)` on this rank's
    shard.  With gather=True returns the full (probs, labels) of all N pairs on every rank, in the
    original pair order; otherwise returns this rank's shard and its [lo, hi)."""
    import torch
    import torch.distributed as dist

    N = int(len(pairs))
    lo, hi = shard_bounds(N, world, rank)
    probs, labels = query_fn(pairs[lo:hi], poses[lo:hi])
    probs = np.asarray(probs, np.float32)
    labels = np.asarray(labels, np.uint8)
    if not gather or world == 1:
        return (probs, labels) if gather else (probs, labels, (lo, hi))
    per = -(-N // world)
    dev = device if device is not None else torch.device("cpu")
    buf = torch.zeros(per, 2, dtype=torch.float32, device=dev)  # (prob, label) per pair, padded
    if hi > lo:
        buf[: hi - lo, 0] = torch.from_numpy(probs).to(dev)
        buf[: hi - lo, 1] = torch.from_numpy(labels.astype(np.float32)).to(dev)
    out = torch.empty(world * per, 2, dtype=torch.float32, device=dev)
    dist.all_gather_into_tensor(out, buf, group=group)
    out = out[:N].cpu().numpy()
    return out[:, 0].copy(), out[:, 1].astype(np.uint8)
