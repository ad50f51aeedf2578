"""Operator-level mask-fused attention on the GPU (reference attention.py:25-217).

Same names, argument meaning and errors as the reference. Inputs may be
numpy arrays (copied to the device, results written back in place, like the
reference's in-place ops) or CUDA tensors (operated on directly).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib
from .core import BatchDescriptor
from .folding import FoldingPlan, plan_folding


def _stream() -> int:
    import torch
    return torch.cuda.current_stream().cuda_stream


def _to_device_f32(a):
    """(cuda float32 contiguous tensor, source-was-numpy flag)."""
    import torch
    if torch.is_tensor(a):
        t = a if a.is_cuda else a.cuda()
        if t.dtype != torch.float32:
            t = t.float()
        return t.contiguous(), False
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).cuda(), True


def _writeback(dst, dev) -> None:
    """Copy a device result into ``dst`` in place (numpy or tensor)."""
    import torch
    if torch.is_tensor(dst):
        if dst.data_ptr() != dev.data_ptr():
            dst.copy_(dev)
    else:
        np.copyto(dst, dev.cpu().numpy())


def _pads_dev(desc: BatchDescriptor):
    import torch
    return torch.tensor(desc.padding_len, dtype=torch.int32, device="cuda")


def _shape(a):
    return tuple(a.shape)


@dataclass
class AttentionScores:
    """Score planes [batch * head_count, query_len, key_len] (attention.py:25-40)."""

    data: object
    batch: int
    head_count: int

    def __post_init__(self):
        shp = _shape(self.data)
        if len(shp) != 3:
            raise ValueError(f"scores must be 3-d, got shape {shp}")
        if shp[0] != self.batch * self.head_count:
            raise ValueError(f"first dimension {shp[0]} != batch {self.batch} x heads {self.head_count}")


def _check_scores(scores: AttentionScores, desc: BatchDescriptor) -> None:
    if scores.batch != desc.batch:
        raise ValueError(f"scores batch {scores.batch} != descriptor batch {desc.batch}")
    shp = _shape(scores.data)
    if shp[1] != desc.seq_len or shp[2] != desc.seq_len:
        raise ValueError(f"score planes {shp[1:]} != (seq_len, seq_len) = ({desc.seq_len}, {desc.seq_len})")


def _plan_for(size: int, plan: FoldingPlan | None, what: str) -> FoldingPlan:
    if plan is None:
        return plan_folding(size)
    if plan.logical_size != size:
        raise ValueError(f"plan covers {plan.logical_size} keys, {what} has {size}")
    return plan


def _masked(scores: AttentionScores, desc: BatchDescriptor, plan, causal: bool) -> AttentionScores:
    _check_scores(scores, desc)
    plan = _plan_for(desc.seq_len, plan, "descriptor")
    dev, _ = _to_device_f32(scores.data)
    _lib.call("eet_masked_softmax", dev.data_ptr(), _pads_dev(desc).data_ptr(), desc.batch,
              scores.head_count, desc.seq_len, 1 if causal else 0, plan.unit_cap, _stream())
    _writeback(scores.data, dev)
    return scores


def fused_causal_softmax(scores: AttentionScores, desc: BatchDescriptor,
                         plan: FoldingPlan | None = None) -> AttentionScores:
    """Causal + padding softmax in place: row i >= pad_b over keys [pad_b, i],
    exact zeros elsewhere and on pad-query rows (attention.py:73-104)."""
    return _masked(scores, desc, plan, True)


def fused_padding_softmax(scores: AttentionScores, desc: BatchDescriptor,
                          plan: FoldingPlan | None = None) -> AttentionScores:
    """Bidirectional padding softmax in place: keys [pad_b, s) (attention.py:107-135)."""
    return _masked(scores, desc, plan, False)


def fused_step_softmax(scores, desc: BatchDescriptor, plan: FoldingPlan | None = None):
    """Decode-step softmax in place over [b, heads, L]: slots [pad_b, L)
    (attention.py:138-163)."""
    b, heads, length = _shape(scores)
    if b != desc.batch:
        raise ValueError(f"scores batch {b} != descriptor batch {desc.batch}")
    plan = _plan_for(length, plan, "scores")
    dev, _ = _to_device_f32(scores)
    _lib.call("eet_step_softmax", dev.data_ptr(), _pads_dev(desc).data_ptr(), b, heads, length,
              plan.unit_cap, _stream())
    _writeback(scores, dev)
    return scores


def split_heads(x, head_count: int):
    """[b, t, h] -> [b, heads, t, head_dim] view."""
    b, t, h = _shape(x)
    r = x.reshape(b, t, head_count, h // head_count)
    return r.transpose(0, 2, 1, 3) if isinstance(r, np.ndarray) else r.permute(0, 2, 1, 3)


def mha_forward(q, k, v, desc: BatchDescriptor, head_count: int, causal: bool = True,
                plan: FoldingPlan | None = None):
    """Scaled dot-product attention with index-derived masks, [b, s, h] in
    and out; pad-query rows zero (attention.py:172-217). One fused kernel:
    no score tensor and no mask tensor are materialised."""
    if _shape(q) != _shape(k) or _shape(q) != _shape(v):
        raise ValueError(f"q/k/v shapes differ: {_shape(q)} {_shape(k)} {_shape(v)}")
    b, t, h = _shape(q)
    if b != desc.batch or t != desc.seq_len:
        raise ValueError(f"inputs [{b}, {t}, ...] do not match descriptor "
                         f"(batch {desc.batch}, seq_len {desc.seq_len})")
    if h % head_count != 0:
        raise ValueError(f"hidden {h} not divisible by {head_count} heads")
    if plan is not None and plan.logical_size != t:
        raise ValueError(f"plan covers {plan.logical_size} keys, inputs have {t}")
    import torch
    qd, from_np = _to_device_f32(q)
    kd, _ = _to_device_f32(k)
    vd, _ = _to_device_f32(v)
    out = torch.empty_like(qd)
    _lib.call("eet_mha_forward", qd.data_ptr(), kd.data_ptr(), vd.data_ptr(), out.data_ptr(),
              _pads_dev(desc).data_ptr(), b, t, h, head_count, 1 if causal else 0, _stream())
    return out.cpu().numpy() if from_np else out
