"""Batch-sharded data parallelism over one process per GPU.

Sequences are independent work items (attention is per (sequence, head)
plane), so a batch is partitioned across ranks with no
collective on the data path: every rank runs ``generate`` on its shard with
its own replicated weights, KV cache and arena, and the tokens are gathered
once at the end. Because each shard runs the same kernels on the same
per-sequence work, every row is bit-identical to the single-GPU result.

Shards balance the causal prompt work (sum over sequences of len^2 + len)
with a deterministic longest-first greedy assignment.
"""

from __future__ import annotations

import numpy as np


def shard_lengths(lengths, world: int) -> list:
    """Sequence indices per rank, longest-first greedy on len*(len+1)."""
    if world < 1:
        raise ValueError("world size must be >= 1")
    cost = [int(n) * (int(n) + 1) for n in lengths]
    order = sorted(range(len(cost)), key=lambda i: (-cost[i], i))
    load = [0] * world
    shards = [[] for _ in range(world)]
    for i in order:
        r = min(range(world), key=lambda k: (load[k], len(shards[k]), k))
        shards[r].append(i)
        load[r] += cost[i]
    return [sorted(s) for s in shards]


def generate_dp(weights, req, cfg, *, group=None, local_generate=None, **kw) -> np.ndarray:
    """``generate`` over the ranks of ``group`` (torch.distributed): each rank
    decodes its shard of ``req.prompts``; returns the full [batch, steps]
    token matrix on every rank. ``local_generate`` defaults to
    :func:`paper_2104_12470_b200.generate` (tests substitute a CPU stub)."""
    import torch.distributed as dist
    from .runtime import GenerationRequest
    if local_generate is None:
        from .runtime import generate as local_generate
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    shards = shard_lengths([len(p) for p in req.prompts], world)
    mine = shards[rank]
    if mine:
        sub = GenerationRequest(prompts=[req.prompts[i] for i in mine], steps=req.steps)
        toks = np.asarray(local_generate(weights, sub, cfg, **kw), dtype=np.int64)
    else:
        toks = np.zeros((0, req.steps), dtype=np.int64)
    gathered = [None] * world
    dist.all_gather_object(gathered, (mine, toks), group=group)
    out = np.zeros((len(req.prompts), req.steps), dtype=np.int64)
    for idx, t in gathered:
        for row, i in enumerate(idx):
            out[i] = t[row]
    return out
