"""Decoder/encoder layers and two-phase generation on the B200 (reference
runtime.py:43-437).

``decoder_layer_forward`` and ``generate`` keep the reference signatures,
validation and error messages; the work happens in one C-ABI call each
(csrc/runtime.cu): the layer is LN -> fused-QKV GEMM (K/V scattered straight
into the cache) -> mask-fused attention -> out-proj GEMM (+residual) -> LN ->
W1 GEMM (+GELU) -> W2 GEMM (+residual), over the packed valid tokens only.
``generate`` runs the prompt pass, then replays a CUDA graph of one decode
step (all layers + LM head + argmax) per generated token.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from enum import Enum

import numpy as np

from . import _lib
from .core import BatchDescriptor, ModelConfig, make_batch, validate_config
from .memory import ActivationCaches, AllocationLog, BufferPool, CacheOverflowError, KVCache, preallocate_caches
from .weights import DeviceLayer, DeviceModel, LayerWeights, ModelWeights


class Phase(Enum):
    PROMPT_PARALLEL = "prompt_parallel"
    INCREMENTAL = "incremental"


@dataclass
class GenerationRequest:
    """Greedy generation of ``steps`` tokens after per-sequence prompts
    (runtime.py:51-69)."""

    prompts: list
    steps: int
    strategy: str = "greedy"

    def __post_init__(self):
        if self.strategy != "greedy":
            raise ValueError(f"unsupported strategy {self.strategy!r}")
        if not self.prompts:
            raise ValueError("request needs at least one prompt")
        if any(len(p) < 1 for p in self.prompts):
            raise ValueError("every prompt must have at least one token")
        if self.steps < 0:
            raise ValueError("steps must be >= 0")


@dataclass
class RunTrace:
    """Work counters and optional per-step logits (runtime.py:72-80)."""

    layer_invocations: int = 0
    prompt_passes: int = 0
    decode_steps: int = 0
    collect_logits: bool = False
    step_logits: list = field(default_factory=list)


def _stream() -> int:
    import torch
    return torch.cuda.current_stream().cuda_stream


def _hidden_on_device(x):
    """Return (float32 CUDA tensor with unit inner stride, needs_writeback)."""
    import torch
    if torch.is_tensor(x) and x.is_cuda and x.dtype == torch.float32 and x.stride(-1) == 1:
        return x, False
    if torch.is_tensor(x):
        return x.detach().to(device="cuda", dtype=torch.float32).contiguous(), True
    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32)).cuda(), True


def _writeback(x, dev):
    import torch
    if torch.is_tensor(x):
        x.copy_(dev)
    else:
        np.copyto(x, dev.cpu().numpy())


def _pads_c(desc: BatchDescriptor):
    return (C.c_int * desc.batch)(*desc.padding_len)


def layer_norm(x, scale, shift, out=None):
    """Row LayerNorm on the GPU (runtime.py:83-94); float32 in and out."""
    import torch
    from .attention import _to_device_f32
    xd, from_np = _to_device_f32(x)
    g, _ = _to_device_f32(scale)
    b, _ = _to_device_f32(shift)
    h = xd.shape[-1]
    y = torch.empty_like(xd)
    _lib.call("eet_layer_norm", xd.data_ptr(), g.data_ptr(), b.data_ptr(), y.data_ptr(),
              xd.numel() // h, h, 0, _stream())
    res = y.cpu().numpy() if from_np else y
    if out is not None:
        _writeback(out, y)
        return out
    return res


def decoder_layer_forward(x, w: LayerWeights, kv: KVCache, desc: BatchDescriptor, phase: Phase,
                          pool: BufferPool, acts: ActivationCaches, layer_idx: int,
                          trace: RunTrace | None = None):
    """One pre-norm decoder layer, in place on ``x`` [b, t, h]
    (runtime.py:217-263). PROMPT_PARALLEL writes K/V for every prompt slot
    and attends causally within the prompt; INCREMENTAL appends one slot and
    attends over the cache. The caller advances the cache cursor."""
    b, t, h = tuple(x.shape)
    if phase is Phase.INCREMENTAL:
        if t != 1:
            raise ValueError(f"incremental step takes 1 token, got {t}")
        if kv.filled < desc.seq_len:
            raise ValueError("incremental phase before the prompt was cached")
    else:
        if t != desc.seq_len:
            raise ValueError(f"prompt pass covers {desc.seq_len} slots, got {t}")
        if kv.filled != 0:
            raise ValueError("prompt phase expects an empty cache")
    if kv.filled + t > kv.max_sequence:
        raise CacheOverflowError(f"step would fill {kv.filled + t} of {kv.max_sequence} cache slots")
    if b != desc.batch:
        raise ValueError(f"scores batch {b} != descriptor batch {desc.batch}")
    cfg = kv.config
    if h != cfg.hidden_size:
        raise ValueError(f"hidden {h} does not match the cache's {cfg.hidden_size}")
    right = getattr(desc, "padding_side", "left") == "right"
    if right and phase is Phase.INCREMENTAL:
        raise ValueError("incremental step needs a left-padded batch (one common cache cursor)")
    dl = DeviceLayer.of(w, kv.dtype)
    rt = pool.runtime(kv.dtype, h, kv.head_count, cfg.batch_size, cfg.max_sequence)
    xd, wb = _hidden_on_device(x)
    ph = _lib.PHASE_INCREMENTAL if phase is Phase.INCREMENTAL else _lib.PHASE_PROMPT
    try:
        if right:                                        # native windows [0, len_b)
            starts, ends = zip(*desc.windows())
            _lib.call("eet_decoder_layer_forward_window", rt, xd.data_ptr(), xd.stride(0), xd.stride(1), b, t,
                      C.byref(dl.c), kv._k[layer_idx].data_ptr(), kv._v[layer_idx].data_ptr(),
                      (C.c_int * b)(*starts), (C.c_int * b)(*ends), _stream())
        else:
            _lib.call("eet_decoder_layer_forward", rt, xd.data_ptr(), xd.stride(0), xd.stride(1), b, t,
                      C.byref(dl.c), kv._k[layer_idx].data_ptr(), kv._v[layer_idx].data_ptr(), kv.filled,
                      _pads_c(desc), desc.seq_len, ph, _stream())
    finally:
        pool._sync_log()
    if wb:
        _writeback(x, xd)
    if trace is not None:
        trace.layer_invocations += 1
    return x


def encoder_layer_forward(x, w: LayerWeights, desc: BatchDescriptor, pool: BufferPool,
                          head_count: int, acts: ActivationCaches | None = None,
                          trace: RunTrace | None = None, datatype_label: str = "fp32"):
    """One pre-norm bidirectional layer, in place (runtime.py:266-301)."""
    from .core import dtype_code
    b, t, h = tuple(x.shape)
    if b != desc.batch or t != desc.seq_len:
        raise ValueError(f"input [{b}, {t}, ...] does not match descriptor "
                         f"(batch {desc.batch}, seq_len {desc.seq_len})")
    if h % head_count != 0:
        raise ValueError(f"hidden {h} not divisible by {head_count} heads")
    dt = dtype_code(datatype_label)
    dl = DeviceLayer.of(w, dt)
    rt = pool.runtime(dt, h, head_count, b, t)
    xd, wb = _hidden_on_device(x)
    try:
        if getattr(desc, "padding_side", "left") == "right":
            starts, ends = zip(*desc.windows())
            _lib.call("eet_encoder_layer_forward_window", rt, xd.data_ptr(), xd.stride(0), xd.stride(1), b, t,
                      C.byref(dl.c), (C.c_int * b)(*starts), (C.c_int * b)(*ends), _stream())
        else:
            _lib.call("eet_encoder_layer_forward", rt, xd.data_ptr(), xd.stride(0), xd.stride(1), b, t,
                      C.byref(dl.c), _pads_c(desc), _stream())
    finally:
        pool._sync_log()
    if wb:
        _writeback(x, xd)
    if trace is not None:
        trace.layer_invocations += 1
    return x


def _validate_request(weights: ModelWeights, req: GenerationRequest, cfg: ModelConfig) -> None:
    """Same checks and messages as runtime.py:347-369."""
    validate_config(cfg)
    if weights.hidden_size != cfg.hidden_size or weights.layer_count != cfg.layer_count:
        raise ValueError("weights do not match the configuration")
    if len(req.prompts) > cfg.batch_size:
        raise ValueError(f"batch {len(req.prompts)} exceeds configured maximum {cfg.batch_size}")
    longest = max(len(p) for p in req.prompts)
    if longest > cfg.max_prompt:
        raise ValueError(f"prompt length {longest} exceeds max prompt {cfg.max_prompt}")
    if longest + req.steps > cfg.max_sequence:
        raise ValueError(f"prompt {longest} + steps {req.steps} exceeds max sequence {cfg.max_sequence}")
    flat = np.concatenate([np.asarray(p, dtype=np.int64) for p in req.prompts])
    bad = flat[(flat < 0) | (flat >= weights.vocab)]
    if bad.size:
        raise ValueError(f"token id {int(bad[0])} outside vocab [0, {weights.vocab})")


def generate(weights: ModelWeights, req: GenerationRequest, cfg: ModelConfig, *,
             pool: BufferPool | None = None, log: AllocationLog | None = None,
             trace: RunTrace | None = None, caches=None, use_graph: bool = True) -> np.ndarray:
    """Greedy decoding: one prompt-parallel pass, then ``req.steps``
    incremental steps (runtime.py:372-437). Returns int64 [batch, steps];
    ties break toward the lowest token id."""
    import torch
    _validate_request(weights, req, cfg)
    if log is None:
        log = AllocationLog()
    if pool is None:
        pool = BufferPool(log=log)
    if caches is None:
        kv, acts = preallocate_caches(cfg, log=log)
    else:
        kv, acts = caches
        if kv.config != cfg or acts.config != cfg:
            raise ValueError("injected caches were built for another configuration")
        if kv.filled != 0:
            raise ValueError("injected K/V cache is not empty")

    nb = len(req.prompts)
    desc = make_batch([len(p) for p in req.prompts])
    t, steps = desc.seq_len, req.steps
    dm = DeviceModel.of(weights, kv.dtype)
    rt = pool.runtime(kv.dtype, cfg.hidden_size, cfg.head_count, cfg.batch_size, cfg.max_sequence)
    prompts = np.zeros((nb, t), dtype=np.int32)
    for i, p in enumerate(req.prompts):
        prompts[i, :len(p)] = p
    lengths = np.asarray([len(p) for p in req.prompts], dtype=np.int32)
    tokens = np.zeros((nb, steps), dtype=np.int64)
    logits = None
    if trace is not None and trace.collect_logits and steps > 0:
        logits = torch.empty((steps, nb, weights.vocab), dtype=torch.float32, device="cuda")
    model, keep = dm.cstruct(kv, acts, cfg.max_prompt)
    try:
        _lib.call("eet_generate", rt, C.byref(model),
                  prompts.ctypes.data_as(C.POINTER(C.c_int)), lengths.ctypes.data_as(C.POINTER(C.c_int)),
                  nb, t, steps, tokens.ctypes.data_as(C.POINTER(C.c_longlong)),
                  logits.data_ptr() if logits is not None else None, 1 if use_graph else 0, _stream())
    finally:
        pool._sync_log()
    kv.advance(t)
    if trace is not None:
        trace.layer_invocations += weights.layer_count * (1 + steps)
        trace.prompt_passes += 1
        trace.decode_steps += steps
        if logits is not None:
            host = logits.cpu().numpy()
            trace.step_logits.extend(host[s].copy() for s in range(steps))
    if steps:
        kv.advance(steps)
    return tokens
