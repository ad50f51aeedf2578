"""CPU restatement (numpy, float32) of the reference decoder-layer path.

TEST INFRASTRUCTURE ONLY (see ``oracle/__init__.py``). Every function cites the
reference ``maskfold`` file:line it restates; paths are relative to
``/root/reference/pkg/src/maskfold/``. The restatement is written independently
(vectorised index-window masks instead of the reference's per-row Python
loops) and is pinned to the real reference by ``tests/golden``.

Numerics: float32 everywhere, like the reference (``core.py:20``). Softmax
normalisers are summed with numpy's pairwise sum rather than the reference's
block-ordered sum (``attention.py:55-66``); both are exact to ~1 ulp, far
inside the reference tests' own 1e-6 tolerance.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

F32 = np.float32
LN_EPS = F32(1e-5)                       # runtime.py:43
GELU_C = F32(math.sqrt(2.0 / math.pi))   # runtime.py:44
GELU_A = F32(0.044715)                   # runtime.py:45

__all__ = [
    "LN_EPS", "layer_norm", "gelu_tanh", "left_pads", "lengths_for_ratio",
    "window_bounds", "masked_softmax", "step_softmax", "mha",
    "OracleKV", "decoder_layer", "encoder_layer", "generate",
    "seeded_weights", "OracleLayer", "OracleModel", "head_logits",
    "decoder_layer_rows",
]


# --------------------------------------------------------------------------
# batch description
# --------------------------------------------------------------------------
def left_pads(lengths, target=None) -> tuple[int, ...]:
    """Max-length left padding: pad_b = target - len_b (core.py:126-146)."""
    lengths = [int(n) for n in lengths]
    if not lengths or min(lengths) < 1:
        raise ValueError("prompt lengths must be non-empty and >= 1")
    target = max(lengths) if target is None else int(target)
    if target < max(lengths):
        raise ValueError("target shorter than the longest prompt")
    return tuple(target - n for n in lengths)


def lengths_for_ratio(batch: int, prompt: int, ratio: float) -> list[int]:
    """Prompt lengths whose pad share approximates ``ratio`` (bench.py:170-191):
    sequence 0 stays full; the pad budget is spread as ceil-shares over the
    remaining sequences, each keeping at least one token."""
    if not 0.0 <= ratio < 1.0:
        raise ValueError("ratio must be in [0, 1)")
    out = [prompt] * batch
    budget = round(ratio * batch * prompt)
    if budget == 0:
        return out
    if batch == 1:
        raise ValueError("a single sequence cannot carry padding")
    for i in range(1, batch):
        take = min(prompt - 1, -(-budget // (batch - i)))
        out[i] = prompt - take
        budget -= take
        if budget <= 0:
            break
    return out


# --------------------------------------------------------------------------
# row ops
# --------------------------------------------------------------------------
def layer_norm(x, gamma, beta):
    """(x - mean) / sqrt(var_pop + eps) * gamma + beta (runtime.py:83-94)."""
    x = np.asarray(x, dtype=F32)
    mu = np.mean(x, axis=-1, keepdims=True)
    var = np.var(x, axis=-1, keepdims=True)
    return ((x - mu) / np.sqrt(var + LN_EPS)) * gamma + beta


def gelu_tanh(u):
    """u * 0.5 * (1 + tanh(c (u + a u^3))) (runtime.py:97-103)."""
    u = np.asarray(u, dtype=F32)
    return u * (F32(0.5) * (F32(1.0) + np.tanh(GELU_C * (u + GELU_A * u * u * u))))


# --------------------------------------------------------------------------
# mask-fused softmax (index-window semantics of attention.py:73-163)
# --------------------------------------------------------------------------
def window_bounds(pad: int, s: int, causal: bool):
    """Boolean [s, s] window: query i >= pad attends keys pad <= j <= i
    (causal, attention.py:88-101) or pad <= j < s (bidirectional,
    attention.py:107-135). Pad-query rows have an empty window."""
    i = np.arange(s)[:, None]
    j = np.arange(s)[None, :]
    win = (i >= pad) & (j >= pad)
    if causal:
        win &= j <= i
    return win


def _softmax_in_window(x, win):
    """Softmax over ``win`` with exact zeros outside and for empty rows."""
    neg = np.where(win, x, F32(-np.inf))
    m = np.max(neg, axis=-1, keepdims=True)
    m = np.where(np.isfinite(m), m, F32(0.0))
    e = np.where(win, np.exp(np.where(win, x - m, F32(0.0))), F32(0.0)).astype(F32)
    tot = np.sum(e, axis=-1, keepdims=True, dtype=F32)
    return (e / np.where(tot > 0, tot, F32(1.0))).astype(F32)


def masked_softmax(scores, pads, heads: int, causal: bool = True):
    """scores [b*heads, s, s] -> new array; ``fused_causal_softmax`` /
    ``fused_padding_softmax`` (attention.py:73-135)."""
    scores = np.asarray(scores, dtype=F32)
    bh, s, s2 = scores.shape
    if s != s2 or bh != len(pads) * heads:
        raise ValueError("score planes do not match the descriptor")
    out = np.empty_like(scores)
    for b, pad in enumerate(pads):
        win = window_bounds(pad, s, causal)
        sl = slice(b * heads, (b + 1) * heads)
        out[sl] = _softmax_in_window(scores[sl], win[None])
    return out


def step_softmax(scores, pads):
    """scores [b, heads, L] -> new array; softmax over slots [pad_b, L),
    zeros below (``fused_step_softmax``, attention.py:138-163)."""
    scores = np.asarray(scores, dtype=F32)
    b, heads, L = scores.shape
    win = np.arange(L)[None, :] >= np.asarray(pads)[:, None]      # [b, L]
    return _softmax_in_window(scores, win[:, None, :])


def mha(q, k, v, pads, heads: int, causal: bool = True):
    """Scaled dot-product attention, [b, s, h] in and out, pad-query rows
    zero (``mha_forward``, attention.py:172-217). Scale is applied after the
    product (attention.py:206-207)."""
    q, k, v = (np.asarray(a, dtype=F32) for a in (q, k, v))
    b, s, h = q.shape
    hd = h // heads

    def split(a):
        return a.reshape(b, s, heads, hd).transpose(0, 2, 1, 3)

    sc = np.matmul(split(q), split(k).transpose(0, 1, 3, 2)).reshape(b * heads, s, s)
    sc = sc * F32(1.0 / math.sqrt(hd))
    p = masked_softmax(sc, pads, heads, causal).reshape(b, heads, s, s)
    ctx = np.matmul(p, split(v))                                    # [b, n, s, hd]
    return np.ascontiguousarray(ctx.transpose(0, 2, 1, 3)).reshape(b, s, h)


# --------------------------------------------------------------------------
# weights (seeded init identical to weights.py:99-139)
# --------------------------------------------------------------------------
@dataclass
class OracleLayer:
    ln1_scale: np.ndarray
    ln1_shift: np.ndarray
    wq: np.ndarray
    wk: np.ndarray
    wv: np.ndarray
    wo: np.ndarray
    ln2_scale: np.ndarray
    ln2_shift: np.ndarray
    w1: np.ndarray
    w2: np.ndarray


@dataclass
class OracleModel:
    hidden_size: int
    head_count: int
    vocab: int
    max_sequence: int
    token_embedding: np.ndarray
    position_embedding: np.ndarray
    layers: list
    final_scale: np.ndarray
    final_shift: np.ndarray
    output_head: np.ndarray


def seeded_weights(hidden, layers, heads, vocab, max_sequence, seed, scale=0.02):
    """N(0, scale^2) float32 weights drawn from ``default_rng(seed)`` in the
    reference order: per layer wq, wk, wv, wo, w1, w2; then token embedding,
    position embedding, output head; LN scales 1, shifts 0
    (weights.py:99-139)."""
    rng = np.random.default_rng(seed)
    h = int(hidden)

    def draw(*shape):
        return rng.normal(0.0, scale, size=shape).astype(F32)

    ones = lambda: np.ones(h, dtype=F32)       # noqa: E731
    zeros = lambda: np.zeros(h, dtype=F32)     # noqa: E731
    lw = []
    for _ in range(layers):
        wq, wk, wv, wo = draw(h, h), draw(h, h), draw(h, h), draw(h, h)
        w1, w2 = draw(h, 4 * h), draw(4 * h, h)
        lw.append(OracleLayer(ones(), zeros(), wq, wk, wv, wo, ones(), zeros(), w1, w2))
    tok = draw(vocab, h)
    pos = draw(max_sequence, h)
    head = draw(h, vocab)
    return OracleModel(h, heads, vocab, max_sequence, tok, pos, lw, ones(), zeros(), head)


# --------------------------------------------------------------------------
# decoder layer with KV cache (runtime.py:106-263, memory.py:237-307)
# --------------------------------------------------------------------------
@dataclass
class OracleKV:
    """Per-layer K/V in [b, n, s_max, hd] with one fill cursor
    (memory.py:237-307)."""

    batch: int
    heads: int
    max_sequence: int
    head_dim: int
    layers: int
    filled: int = 0
    k: list = field(default_factory=list)
    v: list = field(default_factory=list)

    def __post_init__(self):
        shape = (self.batch, self.heads, self.max_sequence, self.head_dim)
        self.k = [np.zeros(shape, F32) for _ in range(self.layers)]
        self.v = [np.zeros(shape, F32) for _ in range(self.layers)]

    def write(self, layer, start, k, v):
        b, t, h = k.shape
        if start + t > self.max_sequence:
            raise OverflowError("cache write past max sequence")
        n, hd = self.heads, self.head_dim
        self.k[layer][:b, :, start:start + t] = k.reshape(b, t, n, hd).transpose(0, 2, 1, 3)
        self.v[layer][:b, :, start:start + t] = v.reshape(b, t, n, hd).transpose(0, 2, 1, 3)

    def advance(self, t):
        if self.filled + t > self.max_sequence:
            raise OverflowError("advance past max sequence")
        self.filled += t


def _attention(x, w, pads, kv: OracleKV | None, layer: int, heads: int, causal: bool):
    """ln1 -> q/k/v -> masked attention -> ctx @ wo (runtime.py:106-189)."""
    b, t, h = x.shape
    hd = h // heads
    ln1 = layer_norm(x, w.ln1_scale, w.ln1_shift)
    q = ln1 @ w.wq
    k = ln1 @ w.wk
    v = ln1 @ w.wv
    qh = q.reshape(b, t, heads, hd).transpose(0, 2, 1, 3)
    scale = F32(1.0 / math.sqrt(hd))
    if kv is None:                                   # encoder (runtime.py:143-153)
        ctx = mha(q, k, v, pads, heads, causal=causal)
        return ctx @ w.wo
    start = kv.filled
    kv.write(layer, start, k, v)
    L = start + t
    kh = kv.k[layer][:b, :, :L]
    vh = kv.v[layer][:b, :, :L]
    sc = np.matmul(qh, kh.transpose(0, 1, 3, 2)) * scale            # [b, n, t, L]
    if t == 1 and start > 0:                         # incremental (runtime.py:155-163)
        p = step_softmax(sc[:, :, 0, :], pads)[:, :, None, :]
    else:                                            # prompt (runtime.py:164-174)
        p = masked_softmax(sc.reshape(b * heads, t, L), pads, heads, True).reshape(b, heads, t, L)
    ctx = np.matmul(p, vh).transpose(0, 2, 1, 3).reshape(b, t, h)   # runtime.py:178
    return ctx @ w.wo                                               # runtime.py:188


def _ffn(x, w):
    """x + gelu(ln2 @ w1) @ w2, accumulated over two 2h chunks like
    runtime.py:192-214."""
    h = x.shape[-1]
    ln2 = layer_norm(x, w.ln2_scale, w.ln2_shift)
    for c0 in (0, 2 * h):
        mid = gelu_tanh(ln2 @ w.w1[:, c0:c0 + 2 * h])
        x = x + mid @ w.w2[c0:c0 + 2 * h, :]
    return x


def decoder_layer(x, w, kv: OracleKV, pads, layer: int, heads: int):
    """One pre-norm decoder layer; returns the new hidden state and writes the
    step's K/V into ``kv`` (the caller advances the cursor), runtime.py:217-263.
    Prompt phase when ``kv.filled == 0``, incremental when t == 1."""
    x = np.asarray(x, dtype=F32)
    t = x.shape[1]
    if kv.filled > 0 and t != 1:
        raise ValueError("incremental step takes 1 token")
    x = x + _attention(x, w, pads, kv, layer, heads, causal=True)
    return _ffn(x, w)


def decoder_layer_rows(x, w, pads, heads: int, rows, kv: OracleKV | None = None, layer: int = 0):
    """Prompt-phase decoder layer (empty cache) evaluated at the query slots
    ``rows`` only: [b, len(rows), h]. Same arithmetic as ``decoder_layer``
    (runtime.py:106-214): K/V come from every slot, but the score plane,
    out-projection and FFN are formed for the selected queries alone, which
    keeps the s=4096 / h=12288 layer shapes within seconds on the host.
    Rows inside a sequence's padding come out as whatever the reference
    computes there (pad-query attention rows are exact zeros,
    attention.py:97-101) and are not compared. With ``kv`` the prompt's K/V
    are written into it (slots [0, t), memory.py:277-292) so incremental
    steps can follow."""
    x = np.asarray(x, dtype=F32)
    b, t, h = x.shape
    hd = h // heads
    rows = np.asarray(rows, dtype=np.int64)
    ln1 = layer_norm(x, w.ln1_scale, w.ln1_shift)
    k = (ln1 @ w.wk).reshape(b, t, heads, hd).transpose(0, 2, 1, 3)
    v = (ln1 @ w.wv).reshape(b, t, heads, hd).transpose(0, 2, 1, 3)
    if kv is not None:
        kv.write(layer, 0, k.transpose(0, 2, 1, 3).reshape(b, t, h), v.transpose(0, 2, 1, 3).reshape(b, t, h))
    q = (ln1[:, rows] @ w.wq).reshape(b, len(rows), heads, hd).transpose(0, 2, 1, 3)
    sc = np.matmul(q, k.transpose(0, 1, 3, 2)) * F32(1.0 / math.sqrt(hd))   # [b, n, r, t]
    p = np.empty_like(sc)
    for i, pad in enumerate(pads):
        win = window_bounds(pad, t, True)[rows]                             # [r, t]
        p[i] = _softmax_in_window(sc[i], win[None])
    ctx = np.matmul(p, v).transpose(0, 2, 1, 3).reshape(b, len(rows), h)
    xr = x[:, rows] + ctx @ w.wo
    return _ffn(xr, w)


def encoder_layer(x, w, pads, heads: int):
    """Bidirectional pre-norm layer (runtime.py:266-301)."""
    x = np.asarray(x, dtype=F32)
    x = x + _attention(x, w, pads, None, 0, heads, causal=False)
    return _ffn(x, w)


# --------------------------------------------------------------------------
# generation (runtime.py:304-437)
# --------------------------------------------------------------------------
def head_logits(model, hid):
    """Final LN + untied output projection (runtime.py:341-344)."""
    return layer_norm(hid, model.final_scale, model.final_shift) @ model.output_head


def generate(model, prompts, steps: int, max_sequence: int | None = None,
             collect_logits: bool = False, layer_limit: int | None = None,
             forced=None):
    """Greedy two-phase generation (runtime.py:372-437). Returns
    (tokens int64 [b, steps], list of per-step logits if requested).

    ``layer_limit`` runs only the first N layers (used by the bounded CPU
    baseline sample; the full path uses every layer). ``forced`` (int
    [b, steps]) teacher-forces the fed-back tokens: step s feeds
    ``forced[:, s]`` instead of the argmax, so per-step logits of another
    implementation can be compared with the reference's at every step even
    after a near-tie picked a different token; the returned tokens are still
    the reference's own argmax."""
    layers = model.layers if layer_limit is None else model.layers[:layer_limit]
    b = len(prompts)
    pads = left_pads([len(p) for p in prompts])
    t = max(len(p) for p in prompts)
    h, n = model.hidden_size, model.head_count
    smax = max_sequence or model.max_sequence
    kv = OracleKV(b, n, smax, h // n, len(layers))
    x = np.zeros((b, t, h), F32)                                  # runtime.py:304-323
    for i, ids in enumerate(prompts):
        x[i, pads[i]:] = model.token_embedding[np.asarray(ids)] + model.position_embedding[:len(ids)]
    for li, w in enumerate(layers):
        x = decoder_layer(x, w, kv, pads, li, n)
    kv.advance(t)
    toks = np.zeros((b, steps), np.int64)
    logs = []
    if steps == 0:
        return toks, logs
    logits = head_logits(model, x[:, -1, :])
    for s in range(steps):
        if collect_logits:
            logs.append(logits.copy())
        nxt = np.argmax(logits, axis=1)                          # lowest id on ties
        toks[:, s] = nxt
        if forced is not None:
            nxt = np.asarray(forced, dtype=np.int64)[:, s]
        pos = (t + s) - np.asarray(pads)                         # runtime.py:326-338
        x1 = (model.token_embedding[nxt] + model.position_embedding[pos])[:, None, :]
        for li, w in enumerate(layers):
            x1 = decoder_layer(x1, w, kv, pads, li, n)
        kv.advance(1)
        logits = head_logits(model, x1[:, 0, :])
    return toks, logs
