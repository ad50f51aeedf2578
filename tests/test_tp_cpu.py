"""Tensor-parallel host logic on CPU: weight sharding + the two all-reduces
per layer, with real gloo collectives over world size 2. Each rank computes
its partial sums with numpy (test-side restatement of the shard math); the
result must equal the oracle's unsharded layer."""

import math
import os
import socket

import numpy as np
import torch.multiprocessing as mp

from paper_2104_12470_b200.tp import shard_config, shard_layer


def _partials(x, w, heads_local, hd):
    from oracle import eet_oracle as orc
    b, t, h = x.shape
    ln1 = orc.layer_norm(x, w.ln1_scale, w.ln1_shift)
    q, k, v = ln1 @ w.wq, ln1 @ w.wk, ln1 @ w.wv                    # [b, t, h/tp]
    ctx = orc.mha(q, k, v, (0,) * b, heads_local, causal=True)
    return ctx @ w.wo                                               # partial [b, t, h]


def _ffn_partial(x, w):
    from oracle import eet_oracle as orc
    ln2 = orc.layer_norm(x, w.ln2_scale, w.ln2_shift)
    return orc.gelu_tanh(ln2 @ w.w1) @ w.w2


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import eet_oracle as orc
    h, heads = 64, 8
    model = orc.seeded_weights(h, 1, heads, 8, 16, seed=5)
    x = np.random.default_rng(1).normal(size=(2, 12, h)).astype(np.float32)
    w = shard_layer(model.layers[0], heads, rank, world)
    p = torch.from_numpy(_partials(x, w, heads // world, h // heads))
    dist.all_reduce(p)
    x = x + p.numpy()
    f = torch.from_numpy(_ffn_partial(x, w))
    dist.all_reduce(f)
    q.put((rank, x + f.numpy()))
    dist.destroy_process_group()


def test_tp2_layer_equals_unsharded_oracle():
    from oracle import eet_oracle as orc
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    h, heads = 64, 8
    model = orc.seeded_weights(h, 1, heads, 8, 16, seed=5)
    x = np.random.default_rng(1).normal(size=(2, 12, h)).astype(np.float32)
    kv = orc.OracleKV(2, heads, 16, h // heads, 1)
    ref = orc.decoder_layer(x, model.layers[0], kv, (0, 0), 0, heads)
    for r in (0, 1):
        np.testing.assert_allclose(res[r], ref, atol=1e-5, rtol=1e-5)


def test_shard_shapes_and_config():
    from oracle import eet_oracle as orc
    import paper_2104_12470_b200 as eet
    model = orc.seeded_weights(96, 1, 12, 8, 16, seed=0)
    for tp in (1, 2, 3, 4):
        parts = [shard_layer(model.layers[0], 12, r, tp) for r in range(tp)]
        assert np.array_equal(np.concatenate([p.wq for p in parts], 1), model.layers[0].wq)
        assert np.array_equal(np.concatenate([p.wo for p in parts], 0), model.layers[0].wo)
        assert np.array_equal(np.concatenate([p.w1 for p in parts], 1), model.layers[0].w1)
        assert np.array_equal(np.concatenate([p.w2 for p in parts], 0), model.layers[0].w2)
    cfg = eet.ModelConfig(2, 96, 1, 12, 8, 16)
    sc = shard_config(cfg, 4)
    assert (sc.head_count, sc.head_dim) == (3, 8)


def test_row_chunks_cover_rows_in_whole_tiles():
    """TensorParallelLayer._chunks: the row-chunked out-proj / W2 (each chunk
    all-reduced while the next one's GEMM runs) covers [0, rows) exactly,
    in order, with chunk boundaries on whole 128-row GEMM tiles."""
    from paper_2104_12470_b200.tp import TensorParallelLayer
    layer = TensorParallelLayer.__new__(TensorParallelLayer)
    for chunks in (0, 1, 3, 4):
        layer.chunks = chunks
        for rows in (1, 100, 128, 255, 256, 1000, 1024, 2048, 15133):
            parts = layer._chunks(rows)
            assert parts[0][0] == 0 and parts[-1][1] == rows
            for (a, b), (c, _) in zip(parts, parts[1:]):
                assert b == c and b % 128 == 0
            assert all(b > a for a, b in parts)
            if chunks:
                assert len(parts) <= chunks
