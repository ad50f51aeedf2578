"""Multi-process product code on one B200 (the only device a gpurun call
has): two ranks share cuda:0 and talk over gloo, so the tensor-parallel and
data-parallel paths run end to end with real collectives.

* TensorParallelLayer.forward (tp = 2, row-chunked out-proj / W2 with the
  all-reduce of each chunk on a side stream; the hook stages the chunk
  through host memory for gloo) — prompt pass + one decode step against
  the unsharded fp32 oracle layer (within tolerance of the
  single-GPU result).
* dp.generate_dp over 2 ranks — every token row bit-identical to the
  single-process generate of the whole batch.

Reference: /root/reference/pkg/src/maskfold/runtime.py:217-263, :372-437.
"""

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _host_all_reduce(t):
    import torch.distributed as dist
    c = t.float().cpu()
    dist.all_reduce(c, op=dist.ReduceOp.SUM)
    t.copy_(c.to(t.dtype))


def _tp_worker(rank, world, port, dt, q):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2104_12470_b200 as eet
        from paper_2104_12470_b200 import _lib
        from paper_2104_12470_b200.tp import TensorParallelLayer, shard_config
        h, heads, lengths = 256, 8, [300, 211, 77]
        desc = eet.make_batch(lengths)
        s, b = desc.seq_len, len(lengths)
        cfg = eet.ModelConfig(batch_size=b, hidden_size=h, layer_count=1, head_count=heads, max_prompt=s,
                              max_sequence=s + 1, datatype_label=dt)
        w = eet.random_weights(cfg, vocab=8, seed=23).layers[0]
        xh = np.random.default_rng(7).normal(0, 1, size=(b, s + 1, h)).astype(np.float32)
        layer = TensorParallelLayer(w, cfg, rank, world, eet.BufferPool(), all_reduce=_host_all_reduce, chunks=3)
        kv = eet.preallocate_caches(shard_config(cfg, world))[0]
        x = torch.from_numpy(xh[:, :s].copy()).cuda()
        layer.forward(x, kv, desc, _lib.PHASE_PROMPT, 0)
        kv.advance(s)
        x1 = torch.from_numpy(xh[:, s:].copy()).cuda()
        layer.forward(x1, kv, desc, _lib.PHASE_INCREMENTAL, 0)
        torch.cuda.synchronize()
        q.put((rank, x.cpu().numpy(), x1.cpu().numpy(), xh, w, desc.padding_len))
    finally:
        dist.destroy_process_group()


def _dp_worker(rank, world, port, q):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2104_12470_b200 as eet
        from paper_2104_12470_b200.dp import generate_dp
        cfg = eet.ModelConfig(batch_size=5, hidden_size=256, layer_count=2, head_count=4, max_prompt=40,
                              max_sequence=48, datatype_label="fp16")
        w = eet.random_weights(cfg, vocab=300, seed=31)
        rng = np.random.default_rng(3)
        prompts = [[int(t) for t in rng.integers(0, 300, size=n)] for n in (40, 13, 29, 7, 33)]
        req = eet.GenerationRequest(prompts=prompts, steps=6)
        toks = generate_dp(w, req, cfg)
        full = eet.generate(w, req, cfg) if rank == 0 else None
        q.put((rank, toks, full))
    finally:
        dist.destroy_process_group()


def _spawn(fn, *args):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=fn, args=(r, 2, port, *args, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = [q.get(timeout=600) for _ in procs]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    return sorted(out, key=lambda r: r[0])


@pytest.mark.parametrize("dt", ["fp32", "bf16"])
def test_tensor_parallel_forward_two_ranks(cuda_ok, dt):
    from conftest import check_16bit, combined_close
    from oracle import eet_oracle as orc
    res = _spawn(_tp_worker, dt)
    (_, x0, s0, xh, w, pads), (_, x1, s1, _, _, _) = res
    assert np.array_equal(x0, x1) and np.array_equal(s0, s1), "ranks disagree on the replicated x"
    b, s = x0.shape[:2]
    heads = 8
    okv = orc.OracleKV(b, heads, s + 1, x0.shape[2] // heads, 1)
    ref = orc.decoder_layer(xh[:, :s], w, okv, pads, 0, heads)
    okv.advance(s)
    ref1 = orc.decoder_layer(xh[:, s:], w, okv, pads, 0, heads)
    for i, pad in enumerate(pads):
        if dt == "fp32":
            combined_close(x0[i, pad:], ref[i, pad:], 1e-5, f"tp2 prompt row {i}")
        else:
            check_16bit(x0[i, pad:], ref[i, pad:], dt, f"tp2 prompt row {i}", emu_ratio=1.0)
    if dt == "fp32":
        combined_close(s0, ref1, 1e-5, "tp2 decode step")
    else:
        check_16bit(s0, ref1, dt, "tp2 decode step", emu_ratio=1.0)


def test_generate_dp_two_ranks_bit_identical(cuda_ok):
    res = _spawn(_dp_worker)
    (_, t0, full), (_, t1, _) = res
    assert np.array_equal(t0, t1)
    assert np.array_equal(t0, full), "data-parallel tokens differ from the single-process generate"
