"""Megatron-style tensor parallelism for the big layers (h 4096-12288,
SURVEY §8(e); new — the reference rejects model parallelism).

Rank r of tp holds heads [r*n/tp, (r+1)*n/tp) of Q/K/V and the matching
rows of Wo, and FFN columns [r*4h/tp, (r+1)*4h/tp) of W1 with the matching
rows of W2. LayerNorm parameters and the residual stream x are replicated. A
layer is two partial products, each summed over ranks (all-reduce) and added
into x:

    x += allreduce(attention_partial(x));   x += allreduce(ffn_partial(x))

The stages are C-ABI calls (``eet_tp_*``, csrc/runtime.cu); the all-reduce
is the communicator's (torch.distributed / NCCL over NVLink by default).
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from .core import BatchDescriptor, ModelConfig
from .memory import BufferPool, KVCache
from .weights import DeviceLayer, LayerWeights


def shard_layer(w: LayerWeights, heads: int, rank: int, tp: int) -> LayerWeights:
    """This rank's slice of one layer's [in, out] weights."""
    h = w.wq.shape[0]
    if heads % tp or (4 * h) % tp:
        raise ValueError(f"heads {heads} and 4*hidden {4 * h} must divide by tp {tp}")
    hq = h // tp                          # = (heads / tp) * head_dim
    q = slice(rank * hq, (rank + 1) * hq)
    f = slice(rank * 4 * h // tp, (rank + 1) * 4 * h // tp)
    return LayerWeights(
        ln1_scale=w.ln1_scale, ln1_shift=w.ln1_shift,
        wq=np.ascontiguousarray(w.wq[:, q]), wk=np.ascontiguousarray(w.wk[:, q]),
        wv=np.ascontiguousarray(w.wv[:, q]), wo=np.ascontiguousarray(w.wo[q, :]),
        ln2_scale=w.ln2_scale, ln2_shift=w.ln2_shift,
        w1=np.ascontiguousarray(w.w1[:, f]), w2=np.ascontiguousarray(w.w2[f, :]))


def shard_config(cfg: ModelConfig, tp: int) -> ModelConfig:
    """Config of this rank's KV cache: heads/tp heads of the same head_dim."""
    return ModelConfig(cfg.batch_size, cfg.hidden_size // tp, cfg.layer_count, cfg.head_count // tp,
                       cfg.max_prompt, cfg.max_sequence, cfg.datatype_label)


def _runtime(pool: BufferPool, dtype: int, hidden: int, heads: int, rank: int, tp: int, bmax: int, smax: int):
    key = ("tp", dtype, hidden, heads, rank, tp, bmax, smax)
    rt = pool._runtimes.get(key)
    if rt is None:
        rt = C.c_void_p()
        _lib.call("eet_runtime_create_tp", C.byref(rt), dtype, hidden, heads, rank, tp, bmax, smax, pool._h)
        pool._runtimes[key] = rt
    return rt


def _default_all_reduce(group):
    def f(t):
        import torch.distributed as dist
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return f


class TensorParallelLayer:
    """One decoder layer sharded over ``tp`` ranks. ``all_reduce(tensor)``
    sums a CUDA tensor over the ranks in place (default: torch.distributed
    on ``group``)."""

    def __init__(self, w: LayerWeights, cfg: ModelConfig, rank: int, tp: int, pool: BufferPool,
                 group=None, all_reduce=None):
        self.cfg, self.rank, self.tp, self.pool = cfg, rank, tp, pool
        self.shard = shard_layer(w, cfg.head_count, rank, tp)
        self.dev = DeviceLayer.of(self.shard, cfg.dtype)
        self.all_reduce = all_reduce or _default_all_reduce(group)
        self.rt = _runtime(pool, cfg.dtype, cfg.hidden_size, cfg.head_count, rank, tp,
                           cfg.batch_size, cfg.max_sequence)

    def attention_partial(self, x, kv: KVCache, desc: BatchDescriptor, phase: int, layer_idx: int):
        import torch
        b, t, h = x.shape
        rows = C.c_int()
        nvalid = b * t - (sum(desc.padding_len) if phase == _lib.PHASE_PROMPT else 0)
        part = torch.empty((max(nvalid, 1), h), dtype=torch.float32, device="cuda")
        _lib.call("eet_tp_attention_partial", self.rt, x.data_ptr(), x.stride(0), x.stride(1), b, t,
                  C.byref(self.dev.c), kv._k[layer_idx].data_ptr(), kv._v[layer_idx].data_ptr(),
                  kv.filled, (C.c_int * b)(*desc.padding_len), desc.seq_len, phase, part.data_ptr(),
                  C.byref(rows), torch.cuda.current_stream().cuda_stream)
        assert rows.value == nvalid
        return part[:nvalid]

    def ffn_partial(self, x):
        import torch
        part = torch.empty((self._rows, x.shape[2]), dtype=torch.float32, device="cuda")
        _lib.call("eet_tp_ffn_partial", self.rt, x.data_ptr(), x.stride(0), x.stride(1),
                  C.byref(self.dev.c), part.data_ptr(), torch.cuda.current_stream().cuda_stream)
        return part

    def residual_add(self, x, reduced):
        import torch
        _lib.call("eet_tp_residual_add", self.rt, x.data_ptr(), x.stride(0), x.stride(1),
                  reduced.data_ptr(), torch.cuda.current_stream().cuda_stream)

    def forward(self, x, kv: KVCache, desc: BatchDescriptor, phase: int, layer_idx: int = 0):
        """decoder_layer_forward (runtime.py:217-263) on this rank's shard;
        x (CUDA float32, replicated) is updated in place on every rank."""
        p = self.attention_partial(x, kv, desc, phase, layer_idx)
        self._rows = p.shape[0]
        self.all_reduce(p)
        self.residual_add(x, p)
        f = self.ffn_partial(x)
        self.all_reduce(f)
        self.residual_add(x, f)
        return x
