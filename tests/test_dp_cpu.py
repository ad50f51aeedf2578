"""Multi-process (world size 2, gloo, CPU) tests of the data-parallel host
logic: shard balancing and the token gather. The per-rank decode is the CPU
oracle here (no GPU); on the GPU box the same code runs the CUDA generate."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2104_12470_b200.dp import generate_dp, shard_lengths


def test_shards_cover_batch_and_balance():
    rng = np.random.default_rng(0)
    for world in (1, 2, 3, 4, 8):
        lengths = [int(v) for v in rng.integers(1, 1025, 32)]
        shards = shard_lengths(lengths, world)
        assert sorted(i for s in shards for i in s) == list(range(32))
        loads = [sum(lengths[i] * (lengths[i] + 1) for i in s) for s in shards]
        assert max(loads) - min(loads) <= max(l * (l + 1) for l in lengths)
    assert shard_lengths([5, 5], 4)[2:] == [[], []]
    with pytest.raises(ValueError):
        shard_lengths([1], 0)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    import torch.distributed as dist
    from oracle import eet_oracle as orc
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2104_12470_b200 as eet
    cfg = eet.ModelConfig(4, 8, 2, 2, 8, 16)
    w = eet.random_weights(cfg, 16, seed=3)
    prompts = [[1, 2, 3], [4, 5, 6, 7, 8], [9], [10, 11]]
    req = eet.GenerationRequest(prompts=prompts, steps=5)

    def local(weights, sub, c):
        toks, _ = orc.generate(weights, sub.prompts, sub.steps, c.max_sequence)
        return toks

    out = generate_dp(w, req, cfg, local_generate=local)
    q.put((rank, out))
    dist.destroy_process_group()


def test_generate_dp_gather_matches_single_process():
    from oracle import eet_oracle as orc
    import paper_2104_12470_b200 as eet
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    cfg = eet.ModelConfig(4, 8, 2, 2, 8, 16)
    w = eet.random_weights(cfg, 16, seed=3)
    # shard decoding is per sequence, so sharded == batched == per-sequence
    single = np.concatenate([orc.generate(w, [p], 5, 16)[0]
                             for p in [[1, 2, 3], [4, 5, 6, 7, 8], [9], [10, 11]]])
    assert np.array_equal(results[0], single)
    assert np.array_equal(results[1], single)
