"""Decoder-layer parity at the BASELINE single-layer shapes (configs 3-5,
SURVEY §8(d)) in bf16 against the fp32 oracle, north-star tolerance 2e-2
(combined form), valid rows only.

The GPU runs the whole configuration; the host oracle checks a subset that
finishes in seconds:
* c3 (h2048, 16 heads, b32, s1024, ragged ``[1024] + rng(3)`` lengths):
  four whole sequences — the reference layer is batch-invariant
  (/root/reference/pkg/tests/test_runtime.py:97-120), so a sequence's output
  does not depend on the other 28 — plus one incremental step.
* c4 (h4096, 32 heads, s4096 = s_max) and c5 (h12288, 96 heads, s2048): a
  spread of query slots through ``oracle.decoder_layer_rows`` (every key,
  selected queries), plus one incremental step for c5. At c5 (K = 4h =
  49152) bf16's own rounding exceeds the elementwise 2e-2 on ~0.8 % of
  elements, so bf16 is held to the norm-wise 2e-2 and to the format's own
  elementwise cost (``conftest.check_16bit``, tests/emu16.py).
* the persistent prefill-attention scheduler's list limit (MAX_ITEMS,
  attn_tc.cu) exceeded, so the per-tile grid fallback runs.

Reference: /root/reference/pkg/src/maskfold/runtime.py:217-263.
"""

import numpy as np
import pytest

from conftest import check_16bit, combined_close

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def eet(cuda_ok):
    import paper_2104_12470_b200 as m
    return m


def _fast_layer(eet, h, seed):
    """N(0, 0.02^2) layer weights drawn with the float32 generator (the
    float64 ``random_weights`` path takes ~1 min at h12288); both sides read
    these same arrays."""
    rng = np.random.default_rng(seed)

    def draw(*shape):
        a = rng.standard_normal(size=shape, dtype=np.float32)
        a *= np.float32(0.02)
        return a

    one, zero = np.ones(h, np.float32), np.zeros(h, np.float32)
    return eet.LayerWeights(one, zero, draw(h, h), draw(h, h), draw(h, h), draw(h, h),
                            one.copy(), zero.copy(), draw(h, 4 * h), draw(4 * h, h))


def _cfg(eet, b, h, heads, p, s, dt="bf16"):
    return eet.ModelConfig(batch_size=b, hidden_size=h, layer_count=1, head_count=heads,
                           max_prompt=p, max_sequence=s, datatype_label=dt)


def _prompt_and_step(eet, w, cfg, desc, x, step_x=None):
    kv, acts = eet.preallocate_caches(cfg)
    pool = eet.BufferPool()
    s = desc.seq_len
    out = eet.decoder_layer_forward(x[:, :s].copy(), w, kv, desc, eet.Phase.PROMPT_PARALLEL, pool, acts, 0)
    st = None
    if step_x is not None:
        kv.advance(s)
        st = eet.decoder_layer_forward(step_x.copy(), w, kv, desc, eet.Phase.INCREMENTAL, pool, acts, 0)
    return out, st


@pytest.mark.parametrize("dt", ["bf16", "fp16"])
def test_c3_ragged_layer(eet, dt):
    from oracle import eet_oracle as orc
    h, heads, s, b = 2048, 16, 1024, 32
    lengths = [1024] + [int(n) for n in np.random.default_rng(3).integers(1, 1025, size=31)]
    desc = eet.make_batch(lengths)
    assert desc.seq_len == s
    w = _fast_layer(eet, h, 30)
    rng = np.random.default_rng(31)
    x = rng.standard_normal(size=(b, s, h), dtype=np.float32)
    step = rng.standard_normal(size=(b, 1, h), dtype=np.float32)
    out, st = _prompt_and_step(eet, w, _cfg(eet, b, h, heads, s, s + 1, dt), desc, x, step)
    ln = np.asarray(lengths)
    pick = sorted({0, int(np.argmin(ln)), int(np.argmax(ln[1:]) + 1),
                   int(np.flatnonzero(ln % 64 != 0)[0])})
    pads = tuple(desc.padding_len[i] for i in pick)
    okv = orc.OracleKV(len(pick), heads, s + 1, h // heads, 1)
    ref = orc.decoder_layer(x[pick], w, okv, pads, 0, heads)
    okv.advance(s)
    ref_st = orc.decoder_layer(step[pick], w, okv, pads, 0, heads)
    for j, i in enumerate(pick):
        combined_close(out[i, pads[j]:], ref[j, pads[j]:], 2e-2, f"c3 {dt} seq {i} (len {lengths[i]})")
    combined_close(st[pick], ref_st, 2e-2, f"c3 {dt} incremental step")


def _rows(s, extra_seed):
    base = {0, 1, 63, 64, 127, 128, 129, 255, 256, s // 2, s - 65, s - 64, s - 2, s - 1}
    base |= {int(r) for r in np.random.default_rng(extra_seed).integers(0, s, size=10)}
    return sorted(r for r in base if 0 <= r < s)


def test_c4_long_context_layer(eet):
    """s = s_max = 4096, plus a ragged second sequence whose valid length is
    not a multiple of the 64-key tile (its last K/V tile ends inside the
    cache plane)."""
    from oracle import eet_oracle as orc
    h, heads, s = 4096, 32, 4096
    lengths = [4096, 3001]
    desc = eet.make_batch(lengths)
    w = _fast_layer(eet, h, 40)
    x = np.random.default_rng(41).standard_normal(size=(2, s, h), dtype=np.float32)
    out, _ = _prompt_and_step(eet, w, _cfg(eet, 2, h, heads, s, s), desc, x)
    rows = _rows(s, 42)
    ref = orc.decoder_layer_rows(x, w, desc.padding_len, heads, rows)
    for i, pad in enumerate(desc.padding_len):
        sel = [j for j, r in enumerate(rows) if r >= pad]
        combined_close(out[i, [rows[j] for j in sel]], ref[i, sel], 2e-2, f"c4 seq {i}")


def test_c5_gpt3_scale_layer(eet):
    from oracle import eet_oracle as orc
    h, heads, s = 12288, 96, 2048
    desc = eet.make_batch([s])
    w = _fast_layer(eet, h, 50)
    rng = np.random.default_rng(51)
    x = rng.standard_normal(size=(1, s, h), dtype=np.float32)
    step = rng.standard_normal(size=(1, 1, h), dtype=np.float32)
    out, st = _prompt_and_step(eet, w, _cfg(eet, 1, h, heads, s, s + 1), desc, x, step)
    rows = _rows(s, 52)
    okv = orc.OracleKV(1, heads, s + 1, h // heads, 1)
    ref = orc.decoder_layer_rows(x, w, desc.padding_len, heads, rows, kv=okv)
    from emu16 import bound_ratio, emu_layer_rows
    emu = bound_ratio(emu_layer_rows(x, w, desc.padding_len, heads, torch.bfloat16, rows)[0], ref[0])
    nr, br = check_16bit(out[0, rows], ref[0], "bf16", "c5 prompt rows", emu)
    print(f"c5 bf16 prompt rows: norm-wise {nr:.4f}, elementwise ratio {br:.3f} (format's own {emu:.3f})")
    okv.advance(s)
    ref_st = orc.decoder_layer(step, w, okv, desc.padding_len, 0, heads)
    check_16bit(st, ref_st, "bf16", "c5 incremental step", emu)


def test_attention_work_list_overflow_falls_back_to_grid(eet):
    """32 sequences x 32 heads x 8 query-tile pairs = 8192 work items > the
    7680-entry list the persistent scheduler passes by value: the per-tile
    grid launch takes over and must agree with the oracle too."""
    from oracle import eet_oracle as orc
    h, heads, s, b = 2048, 32, 2048, 32
    lengths = [2048] + [int(n) for n in np.random.default_rng(6).integers(1800, 2049, size=b - 1)]
    desc = eet.make_batch(lengths)
    w = _fast_layer(eet, h, 60)
    x = np.random.default_rng(61).standard_normal(size=(b, s, h), dtype=np.float32)
    out, _ = _prompt_and_step(eet, w, _cfg(eet, b, h, heads, s, s), desc, x)
    pick = [0, int(np.argmin(lengths))]
    pads = tuple(desc.padding_len[i] for i in pick)
    rows = _rows(s, 62)
    ref = orc.decoder_layer_rows(x[pick], w, pads, heads, rows)
    for j, i in enumerate(pick):
        sel = [k for k, r in enumerate(rows) if r >= pads[j]]
        combined_close(out[i, [rows[k] for k in sel]], ref[j, sel], 2e-2, f"grid fallback seq {i}")
