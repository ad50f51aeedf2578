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
Partials travel in the layer dtype in the 16-bit modes (fp32 in fp32 mode),
and the row-split projections (out-proj, W2) run in row chunks: the
all-reduce of chunk c (on a communication stream) overlaps the GEMM of
chunk c + 1.
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
    on ``group``); it is called on a side stream, once per row chunk."""

    def __init__(self, w: LayerWeights, cfg: ModelConfig, rank: int, tp: int, pool: BufferPool,
                 group=None, all_reduce=None, chunks: int = 0):
        self.cfg, self.rank, self.tp, self.pool = cfg, rank, tp, pool
        self.chunks = chunks                  # row chunks of the overlapped all-reduce (0: by size)
        self._comm = None
        self.shard = shard_layer(w, cfg.head_count, rank, tp)
        self.dev = DeviceLayer.of(self.shard, cfg.dtype)
        self.all_reduce = all_reduce or _default_all_reduce(group)
        self.rt = _runtime(pool, cfg.dtype, cfg.hidden_size, cfg.head_count, rank, tp,
                           cfg.batch_size, cfg.max_sequence)

    def _partial(self, rows, h):
        import torch
        from .memory import torch_dtype
        return torch.empty((max(rows, 1), h), dtype=torch_dtype(self.cfg.dtype), device="cuda")

    def attention_partial(self, x, kv: KVCache, desc: BatchDescriptor, phase: int, layer_idx: int):
        """Whole-layer attention partial (no chunking)."""
        import torch
        b, t, h = x.shape
        rows = C.c_int()
        nvalid = b * t - (sum(desc.padding_len) if phase == _lib.PHASE_PROMPT else 0)
        part = self._partial(nvalid, h)
        _lib.call("eet_tp_attention_partial", self.rt, x.data_ptr(), x.stride(0), x.stride(1), b, t,
                  C.byref(self.dev.c), kv._k[layer_idx].data_ptr(), kv._v[layer_idx].data_ptr(),
                  kv.filled, (C.c_int * b)(*desc.padding_len), desc.seq_len, phase, part.data_ptr(),
                  C.byref(rows), torch.cuda.current_stream().cuda_stream)
        assert rows.value == nvalid
        self._rows = nvalid
        return part[:nvalid]

    def ffn_partial(self, x):
        import torch
        part = self._partial(self._rows, x.shape[2])
        _lib.call("eet_tp_ffn_partial", self.rt, x.data_ptr(), x.stride(0), x.stride(1),
                  C.byref(self.dev.c), part.data_ptr(), torch.cuda.current_stream().cuda_stream)
        return part[:self._rows]

    def residual_add(self, x, reduced):
        import torch
        _lib.call("eet_tp_residual_add", self.rt, x.data_ptr(), x.stride(0), x.stride(1),
                  reduced.data_ptr(), torch.cuda.current_stream().cuda_stream)

    def _chunks(self, rows):
        n = self.chunks if self.chunks else (4 if rows >= 1024 else 2 if rows >= 256 else 1)
        step = -(-rows // n)
        step = -(-step // 128) * 128                    # whole 128-row GEMM tiles per chunk
        return [(r, min(rows, r + step)) for r in range(0, rows, step)]

    def _reduced_rows(self, part, rows, out_rows):
        """out_rows(r0, r1, ptr) computes partial rows on the compute stream;
        each chunk is all-reduced on the communication stream as soon as it
        is written, overlapping the next chunk's GEMM."""
        import torch
        cur = torch.cuda.current_stream()
        if self._comm is None:
            self._comm = torch.cuda.Stream()
        es = part.element_size()
        h = part.shape[1]
        for r0, r1 in self._chunks(rows):
            out_rows(r0, r1, part.data_ptr() + r0 * h * es)
            ev = torch.cuda.Event()
            ev.record(cur)
            self._comm.wait_event(ev)
            with torch.cuda.stream(self._comm):
                self.all_reduce(part[r0:r1])
        cur.wait_stream(self._comm)
        return part[:rows]

    def forward(self, x, kv: KVCache, desc: BatchDescriptor, phase: int, layer_idx: int = 0):
        """decoder_layer_forward (runtime.py:217-263) on this rank's shard;
        x (CUDA float32, replicated) is updated in place on every rank."""
        import torch
        b, t, h = x.shape
        st = lambda: torch.cuda.current_stream().cuda_stream  # noqa: E731
        rows = C.c_int()
        _lib.call("eet_tp_attention_core", self.rt, x.data_ptr(), x.stride(0), x.stride(1), b, t,
                  C.byref(self.dev.c), kv._k[layer_idx].data_ptr(), kv._v[layer_idx].data_ptr(),
                  kv.filled, (C.c_int * b)(*desc.padding_len), desc.seq_len, phase, C.byref(rows), st())
        T = rows.value
        self._rows = T
        part = self._partial(T, h)
        p = self._reduced_rows(part, T, lambda r0, r1, ptr: _lib.call(
            "eet_tp_attention_out", self.rt, C.byref(self.dev.c), r0, r1, ptr, st()))
        self.residual_add(x, p)
        _lib.call("eet_tp_ffn_mid", self.rt, x.data_ptr(), x.stride(0), x.stride(1), C.byref(self.dev.c), st())
        f = self._reduced_rows(part, T, lambda r0, r1, ptr: _lib.call(
            "eet_tp_ffn_out", self.rt, C.byref(self.dev.c), r0, r1, ptr, st()))
        self.residual_add(x, f)
        return x
