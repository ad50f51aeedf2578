"""Weights: host containers, seeded init, MFW1 blob I/O (reference
weights.py:26-204) and their one-time upload to the B200 layout.

Device layout (csrc/ kernels): every projection is stored K-major — the
reference's ``x @ W`` with W [in, out] becomes ``x · Wᵀ`` with Wᵀ [out, in] —
so both tcgen05 operands are K-major and TMA-tileable. Q/K/V are fused into
one [3h, h] matrix (one GEMM per layer instead of three, runtime.py:131,136).
Embeddings and the LM head are stored in the layer dtype; LayerNorm
parameters stay float32.
"""

from __future__ import annotations

import ctypes as C
import struct
from dataclasses import dataclass

import numpy as np

from . import _lib
from .core import FLOAT, ModelConfig, make_tensor, validate_config

MAGIC = b"MFW1"
VERSION = 1
_HEADER = struct.Struct("<6I")       # version, hidden, layers, heads, vocab, max_seq

_LAYER_FIELDS = ("ln1_scale", "ln1_shift", "wq", "wk", "wv", "wo",
                 "ln2_scale", "ln2_shift", "w1", "w2")


@dataclass
class LayerWeights:
    ln1_scale: np.ndarray
    ln1_shift: np.ndarray
    wq: np.ndarray
    wk: np.ndarray
    wv: np.ndarray
    wo: np.ndarray
    ln2_scale: np.ndarray
    ln2_shift: np.ndarray
    w1: np.ndarray  # [h, 4h]
    w2: np.ndarray  # [4h, h]

    def arrays(self) -> list:
        return [getattr(self, f) for f in _LAYER_FIELDS]

    def element_count(self) -> int:
        return sum(a.size for a in self.arrays())


@dataclass
class ModelWeights:
    hidden_size: int
    head_count: int
    vocab: int
    max_sequence: int
    token_embedding: np.ndarray      # [vocab, h]
    position_embedding: np.ndarray   # [max_sequence, h]
    layers: list
    final_scale: np.ndarray
    final_shift: np.ndarray
    output_head: np.ndarray          # [h, vocab]

    @property
    def layer_count(self) -> int:
        return len(self.layers)

    def arrays(self) -> list:
        out = [self.token_embedding, self.position_embedding]
        for lw in self.layers:
            out += lw.arrays()
        return out + [self.final_scale, self.final_shift, self.output_head]

    def element_count(self) -> int:
        return sum(a.size for a in self.arrays())

    def nbytes(self) -> int:
        return self.element_count() * FLOAT().itemsize


def weight_elements(cfg: ModelConfig, vocab: int) -> int:
    h, l = cfg.hidden_size, cfg.layer_count
    return vocab * h + cfg.max_sequence * h + l * (12 * h * h + 4 * h) + 2 * h + h * vocab


def _layer_shapes(h: int):
    return [(h,), (h,), (h, h), (h, h), (h, h), (h, h), (h,), (h,), (h, 4 * h), (4 * h, h)]


def random_weights(cfg: ModelConfig, vocab: int, seed: int, scale: float = 0.02) -> ModelWeights:
    """Seeded N(0, scale^2) float32 weights, drawn in the reference order
    (weights.py:99-139) so both implementations see identical arrays."""
    validate_config(cfg)
    if vocab < 2:
        raise ValueError(f"vocab must be >= 2, got {vocab}")
    rng = np.random.default_rng(seed)
    h = cfg.hidden_size

    def draw(*shape):
        return rng.normal(0.0, scale, size=shape).astype(FLOAT)

    layers = []
    for _ in range(cfg.layer_count):
        wq, wk, wv, wo = (draw(h, h) for _ in range(4))
        w1, w2 = draw(h, 4 * h), draw(4 * h, h)
        layers.append(LayerWeights(np.ones(h, FLOAT), np.zeros(h, FLOAT), wq, wk, wv, wo,
                                   np.ones(h, FLOAT), np.zeros(h, FLOAT), w1, w2))
    tok = draw(vocab, h)
    pos = draw(cfg.max_sequence, h)
    head = draw(h, vocab)
    return ModelWeights(h, cfg.head_count, vocab, cfg.max_sequence, tok, pos, layers,
                        np.ones(h, FLOAT), np.zeros(h, FLOAT), head)


def save_weights(weights: ModelWeights, path) -> None:
    """MFW1 blob (weights.py:142-155, pkg/README.md:107-127)."""
    with open(path, "wb") as fh:
        fh.write(MAGIC)
        fh.write(_HEADER.pack(VERSION, weights.hidden_size, weights.layer_count,
                              weights.head_count, weights.vocab, weights.max_sequence))
        for a in weights.arrays():
            fh.write(np.ascontiguousarray(a, dtype="<f4").tobytes())


def load_weights(path) -> ModelWeights:
    """Parse an MFW1 blob; validates magic, version and exact length
    (weights.py:158-204)."""
    with open(path, "rb") as fh:
        raw = fh.read()
    if raw[:4] != MAGIC:
        raise ValueError(f"bad magic {raw[:4]!r}, expected {MAGIC!r}")
    version, h, nl, heads, vocab, max_seq = _HEADER.unpack(raw[4:4 + _HEADER.size])
    if version != VERSION:
        raise ValueError(f"unsupported blob version {version}")
    payload = np.frombuffer(raw[4 + _HEADER.size:], dtype="<f4")
    shapes = [(vocab, h), (max_seq, h)] + _layer_shapes(h) * nl + [(h,), (h,), (h, vocab)]
    need = sum(int(np.prod(s)) for s in shapes)
    if payload.size < need:
        raise ValueError("weight blob truncated")
    if payload.size > need:
        raise ValueError(f"{payload.size - need} trailing floats in weight blob")
    arrays, off = [], 0
    for s in shapes:
        n = int(np.prod(s))
        arrays.append(make_tensor(s, payload[off:off + n]))
        off += n
    layers = [LayerWeights(*arrays[2 + 10 * i: 12 + 10 * i]) for i in range(nl)]
    return ModelWeights(h, heads, vocab, max_seq, arrays[0], arrays[1], layers,
                        arrays[-3], arrays[-2], arrays[-1])


def load_weights_device(path) -> ModelWeights:
    """MFW1 blob straight to the device (same validation as
    ``load_weights``): the payload is read into pinned host memory, copied to
    HBM in one transfer, and the returned ``ModelWeights`` holds float32 CUDA
    views of it. ``DeviceLayer`` / ``DeviceModel`` then build the K-major
    compute layout with the native transpose+cast kernel
    (``eet_transpose_cast``) -- no host-side transposes or per-array copies."""
    import torch
    with open(path, "rb") as fh:
        head = fh.read(4 + _HEADER.size)
        if head[:4] != MAGIC:
            raise ValueError(f"bad magic {head[:4]!r}, expected {MAGIC!r}")
        if len(head) < 4 + _HEADER.size:
            raise ValueError("weight blob truncated")
        version, h, nl, heads, vocab, max_seq = _HEADER.unpack(head[4:])
        if version != VERSION:
            raise ValueError(f"unsupported blob version {version}")
        shapes = [(vocab, h), (max_seq, h)] + _layer_shapes(h) * nl + [(h,), (h,), (h, vocab)]
        need = sum(int(np.prod(s)) for s in shapes)
        fh.seek(0, 2)
        have = (fh.tell() - 4 - _HEADER.size)
        if have % 4:
            raise ValueError("weight blob length is not a whole number of floats")
        have //= 4
        if have < need:
            raise ValueError("weight blob truncated")
        if have > need:
            raise ValueError(f"{have - need} trailing floats in weight blob")
        host = torch.empty(need, dtype=torch.float32, pin_memory=True)
        fh.seek(4 + _HEADER.size)
        fh.readinto(host.numpy().view(np.uint8))
    dev = host.to("cuda", non_blocking=True)
    torch.cuda.current_stream().synchronize()          # host staging buffer is released below
    del host
    arrays, off = [], 0
    for s in shapes:
        n = int(np.prod(s))
        arrays.append(dev[off:off + n].view(*s))
        off += n
    layers = [LayerWeights(*arrays[2 + 10 * i: 12 + 10 * i]) for i in range(nl)]
    return ModelWeights(h, heads, vocab, max_seq, arrays[0], arrays[1], layers,
                        arrays[-3], arrays[-2], arrays[-1])


# ------------------------------------------------------------------ device
def _is_dev(a) -> bool:
    try:
        import torch
    except ImportError:                                    # pragma: no cover
        return False
    return isinstance(a, torch.Tensor) and a.is_cuda


def _dev(a, dtype):
    import torch
    if _is_dev(a):
        return a.to(dtype=dtype).contiguous()
    return torch.as_tensor(np.ascontiguousarray(a, dtype=np.float32)).to(device="cuda", dtype=dtype).contiguous()


def _dev_t(mats, dtype_code: int, td):
    """Row-stack of the transposes of ``mats`` (each [in, out]) in the
    compute dtype: [sum(out), in]. Device-resident float32 inputs go through
    the native transpose+cast kernel; host arrays through numpy."""
    import torch
    if all(_is_dev(m) for m in mats):
        rows = mats[0].shape[0]
        if any(m.shape[0] != rows for m in mats):
            raise ValueError("stacked matrices need the same input width")
        out = torch.empty((sum(int(m.shape[1]) for m in mats), rows), dtype=td, device="cuda")
        r0 = 0
        for m in mats:
            m = m.to(torch.float32).contiguous()
            cols = int(m.shape[1])
            _lib.call("eet_transpose_cast", dtype_code, m.data_ptr(), rows, cols, out[r0:r0 + cols].data_ptr(),
                      torch.cuda.current_stream().cuda_stream)
            r0 += cols
        return out
    host = mats[0] if len(mats) == 1 else np.concatenate([np.asarray(m) for m in mats], axis=1)
    return _dev(np.asarray(host).T, td)


def _ptr(t) -> int | None:
    return None if t is None else t.data_ptr()


def _fingerprint(arrays) -> tuple:
    """Identity + version of the source arrays behind a cached device upload:
    object id and shape of every array, torch's in-place version counter for
    tensors, and 4 sampled elements of every numpy array (first, thirds,
    last; an in-place write that touches none of them goes unseen: call
    ``invalidate_device_cache`` after editing weights in place). ~1 us per
    array: it runs on every forward."""
    fp = []
    for a in arrays:
        if a is None:
            fp.append(None)
            continue
        if hasattr(a, "_version"):                       # torch tensor
            fp.append((id(a), tuple(a.shape), int(a._version)))
            continue
        n = a.size
        fp.append((id(a), a.shape) + ((a.item(0), a.item(n // 3), a.item(2 * n // 3), a.item(n - 1)) if n else ()))
    return tuple(fp)


def invalidate_device_cache(w) -> None:
    """Drop the device copies cached on a LayerWeights / ModelWeights (and
    its layers): the next forward / generate uploads the arrays again."""
    w.__dict__.pop("_eet_device", None)
    for lw in getattr(w, "layers", []) or []:
        lw.__dict__.pop("_eet_device", None)


class DeviceLayer:
    """One layer's weights in the kernel layout, plus the C struct."""

    def __init__(self, w: LayerWeights, dtype_code: int, biases=None):
        import torch
        from .memory import torch_dtype
        td = torch_dtype(dtype_code)
        f32 = torch.float32
        self.dtype = dtype_code
        self.ln1_g, self.ln1_b = _dev(w.ln1_scale, f32), _dev(w.ln1_shift, f32)
        self.ln2_g, self.ln2_b = _dev(w.ln2_scale, f32), _dev(w.ln2_shift, f32)
        self.wqkv = _dev_t([w.wq, w.wk, w.wv], dtype_code, td)   # [3h, h]
        self.wo = _dev_t([w.wo], dtype_code, td)                   # [h, h]
        self.w1 = _dev_t([w.w1], dtype_code, td)                   # [4h, h]
        self.w2 = _dev_t([w.w2], dtype_code, td)                   # [h, 4h]
        b = biases or {}
        self.b_qkv = _dev(b["qkv"], f32) if "qkv" in b else None
        self.b_o = _dev(b["o"], f32) if "o" in b else None
        self.b_1 = _dev(b["1"], f32) if "1" in b else None
        self.b_2 = _dev(b["2"], f32) if "2" in b else None
        self.c = _lib.LayerWeightsC(
            _ptr(self.ln1_g), _ptr(self.ln1_b), _ptr(self.wqkv), _ptr(self.wo),
            _ptr(self.ln2_g), _ptr(self.ln2_b), _ptr(self.w1), _ptr(self.w2),
            _ptr(self.b_qkv), _ptr(self.b_o), _ptr(self.b_1), _ptr(self.b_2))

    @classmethod
    def of(cls, w: LayerWeights, dtype_code: int) -> "DeviceLayer":
        """Upload once per (weights object, dtype, source-array fingerprint);
        cached on the object. The reference reads its arrays on every call
        (runtime.py:131-212): a replaced or (sampled) modified array uploads
        again instead of serving stale device weights."""
        cache = w.__dict__.setdefault("_eet_device", {})
        fp = _fingerprint(w.arrays())
        hit = cache.get(dtype_code)
        if hit is None or hit[0] != fp:
            hit = cache[dtype_code] = (fp, cls(w, dtype_code))
        return hit[1]


class DeviceModel:
    """Whole model on the device: layers, embeddings, final LN, LM head."""

    def __init__(self, w: ModelWeights, dtype_code: int):
        import torch
        from .memory import torch_dtype
        td = torch_dtype(dtype_code)
        self.dtype = dtype_code
        self.layers = [DeviceLayer.of(lw, dtype_code) for lw in w.layers]
        self.tok = _dev(w.token_embedding, td)
        self.pos = _dev(w.position_embedding, td)
        self.lnf_g = _dev(w.final_scale, torch.float32)
        self.lnf_b = _dev(w.final_shift, torch.float32)
        self.head = _dev_t([w.output_head], dtype_code, td)  # [vocab, h]
        self.vocab = w.vocab
        self.max_sequence = w.max_sequence
        arr = _lib.LayerWeightsC * max(1, len(self.layers))
        self.layer_array = arr(*[dl.c for dl in self.layers])

    @classmethod
    def of(cls, w: ModelWeights, dtype_code: int) -> "DeviceModel":
        """As DeviceLayer.of: keyed on the fingerprint of every array."""
        cache = w.__dict__.setdefault("_eet_device", {})
        fp = _fingerprint(w.arrays()) + (id(w.layers), len(w.layers))
        hit = cache.get(dtype_code)
        if hit is None or hit[0] != fp:
            hit = cache[dtype_code] = (fp, cls(w, dtype_code))
        return hit[1]

    def cstruct(self, kv, acts, max_prompt: int):
        n = len(self.layers)
        kp = (C.c_void_p * max(1, n))(*[t.data_ptr() for t in kv._k])
        vp = (C.c_void_p * max(1, n))(*[t.data_ptr() for t in kv._v])
        m = _lib.ModelC(n, self.vocab, self.max_sequence, self.tok.data_ptr(), self.pos.data_ptr(),
                        C.cast(self.layer_array, C.POINTER(_lib.LayerWeightsC)),
                        self.lnf_g.data_ptr(), self.lnf_b.data_ptr(), self.head.data_ptr(),
                        C.cast(kp, C.POINTER(C.c_void_p)), C.cast(vp, C.POINTER(C.c_void_p)),
                        acts.hidden.data_ptr(), max_prompt)
        return m, (kp, vp)          # keep the pointer arrays alive with the struct
