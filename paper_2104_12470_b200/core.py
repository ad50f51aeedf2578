"""Configuration, tensor and batch-description types (reference core.py:17-146).

Same names, fields and error behaviour as the reference. One extension:
``ModelConfig.datatype_label`` selects the execution dtype of the CUDA path
("fp32" — the reference's numerics, default; "bf16"; "fp16"). The reference
records it as informational only (core.py:62).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

MAX_HIDDEN = 16384      # hidden sizes the folded kernels support (core.py:17)
MAX_SEQUENCE = 4096     # sequence lengths (core.py:18)
FLOAT = np.float32

DTYPES = {"fp32": 0, "float32": 0, "bf16": 1, "bfloat16": 1, "fp16": 2, "float16": 2}


class ConfigError(ValueError):
    """A model configuration violates one of its invariants."""


def dtype_code(label: str) -> int:
    try:
        return DTYPES[label.lower()]
    except KeyError:
        raise ConfigError(f"unsupported datatype_label {label!r}; use one of {sorted(DTYPES)}") from None


def make_tensor(shape, data) -> np.ndarray:
    """Dense row-major float32 tensor of ``shape`` from flat ``data``
    (core.py:27-45): every dim >= 1, element count must match."""
    dims = tuple(int(d) for d in shape)
    if len(dims) == 0:
        raise ValueError("tensor shape must have at least one dimension")
    if min(dims) < 1:
        raise ValueError(f"all dimensions must be >= 1, got {dims}")
    flat = np.ascontiguousarray(data, dtype=FLOAT).ravel()
    if flat.size != math.prod(dims):
        raise ValueError(f"shape {dims} requires {math.prod(dims)} elements, got {flat.size}")
    return flat.reshape(dims)


@dataclass(frozen=True)
class ModelConfig:
    """Capacities of a decoder/encoder stack (b, h, l, heads, p, s)."""

    batch_size: int
    hidden_size: int
    layer_count: int
    head_count: int
    max_prompt: int
    max_sequence: int
    datatype_label: str = "fp32"

    @property
    def head_dim(self) -> int:
        return self.hidden_size // self.head_count

    @property
    def dtype(self) -> int:
        return dtype_code(self.datatype_label)


_RULES = (
    (lambda c: c.batch_size >= 1, lambda c: "batch size must be >= 1"),
    (lambda c: c.hidden_size >= 1, lambda c: "hidden size must be >= 1"),
    (lambda c: c.layer_count >= 0, lambda c: "layer count must be >= 0"),
    (lambda c: c.head_count >= 1, lambda c: "head count must be >= 1"),
    (lambda c: c.max_prompt >= 1, lambda c: "max prompt must be >= 1"),
    (lambda c: c.hidden_size % c.head_count == 0,
     lambda c: f"hidden not divisible by heads ({c.hidden_size} % {c.head_count} != 0)"),
    (lambda c: c.max_prompt <= c.max_sequence,
     lambda c: f"max prompt {c.max_prompt} exceeds max sequence {c.max_sequence}"),
    (lambda c: c.hidden_size <= MAX_HIDDEN,
     lambda c: f"hidden exceeds {MAX_HIDDEN} (got {c.hidden_size})"),
    (lambda c: c.max_sequence <= MAX_SEQUENCE,
     lambda c: f"max sequence exceeds {MAX_SEQUENCE} (got {c.max_sequence})"),
)


def validate_config(cfg: ModelConfig) -> ModelConfig:
    """Raise ConfigError naming the first violated invariant (core.py:69-95)."""
    for ok, msg in _RULES:
        if not ok(cfg):
            raise ConfigError(msg(cfg))
    dtype_code(cfg.datatype_label)
    return cfg


@dataclass(frozen=True)
class BatchDescriptor:
    """Uneven batch (core.py:98-123): left-padded as in the reference —
    sequence i's pads occupy [0, padding_len[i]) — or, new here
    (``padding_side="right"``, BASELINE c1), right-padded:
    its pads occupy [seq_len - padding_len[i], seq_len). A right-padded batch
    runs the prompt pass natively (valid windows, nothing re-laid); the
    incremental phase needs the reference's left padding."""

    seq_len: int
    padding_len: tuple
    batch: int
    padding_side: str = "left"

    def __post_init__(self):
        if self.batch < 1:
            raise ValueError("batch must be >= 1")
        if len(self.padding_len) != self.batch:
            raise ValueError(f"padding_len has {len(self.padding_len)} entries for batch {self.batch}")
        bad = [i for i, p in enumerate(self.padding_len) if not 0 <= p < self.seq_len]
        if bad:
            i = bad[0]
            raise ValueError(f"padding_len[{i}]={self.padding_len[i]} outside [0, {self.seq_len})")
        if self.padding_side not in ("left", "right"):
            raise ValueError(f"padding_side must be 'left' or 'right', got {self.padding_side!r}")

    def pads_array(self) -> np.ndarray:
        return np.asarray(self.padding_len, dtype=np.int32)

    def windows(self):
        """(start, end) of every sequence's valid slots."""
        if self.padding_side == "right":
            return [(0, self.seq_len - p) for p in self.padding_len]
        return [(p, self.seq_len) for p in self.padding_len]


def make_batch(prompt_lengths, target_len: int | None = None, padding_side: str = "left") -> BatchDescriptor:
    """Max-length strategy (core.py:126-146): pad every prompt on the left
    (the reference) or, with ``padding_side="right"``, on the right, to
    ``target_len`` (default: the longest prompt)."""
    lengths = [int(n) for n in prompt_lengths]
    if not lengths:
        raise ValueError("prompt_lengths must not be empty")
    if min(lengths) < 1:
        raise ValueError("every prompt length must be >= 1")
    target = max(lengths) if target_len is None else int(target_len)
    if target < max(lengths):
        raise ValueError(f"target_len {target} shorter than longest prompt {max(lengths)}")
    return BatchDescriptor(seq_len=target, padding_len=tuple(target - n for n in lengths),
                           batch=len(lengths), padding_side=padding_side)
