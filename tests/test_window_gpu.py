"""Right-padded batches (BASELINE configs[0] says "right-padding"; SURVEY
App. B.1): the prompt pass runs natively on per-sequence valid windows
[0, len_b) (``make_batch(..., padding_side="right")`` ->
``eet_decoder_layer_forward_window``), nothing is re-laid.

Oracle: the reference layer is batch-invariant
(/root/reference/pkg/tests/test_runtime.py:97-120), so sequence b of a
right-padded batch must equal the oracle run on its len_b valid rows alone
(runtime.py:217-263; encoder: runtime.py:266-301). fp32 at the north-star
1e-5 (combined form), 16-bit at 2e-2; the 16-bit runs start from a
NaN-filled cache (the tensor-core attention's last K/V tile reaches past a
short sequence's end into slots this pass never writes).
"""

import numpy as np
import pytest

from conftest import combined_close

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def eet(cuda_ok):
    import paper_2104_12470_b200 as m
    return m


CASES = [
    # dtype, hidden, heads, lengths
    ("fp32", 768, 12, [64, 47, 47, 47]),      # BASELINE c1 shape, pad ratio 0.2
    ("fp32", 64, 4, [12, 5, 9]),
    ("bf16", 768, 12, [64, 47, 47, 47]),
    ("fp16", 1024, 16, [300, 77, 129, 1]),     # ends inside and on 64-key tiles
    ("bf16", 512, 4, [256, 190, 64, 200]),     # hd 128
]


@pytest.mark.parametrize("dt,h,heads,lengths", CASES)
def test_right_padded_decoder_layer(eet, dt, h, heads, lengths):
    from oracle import eet_oracle as orc
    desc = eet.make_batch(lengths, padding_side="right")
    s, b = desc.seq_len, len(lengths)
    cfg = eet.ModelConfig(batch_size=b, hidden_size=h, layer_count=1, head_count=heads, max_prompt=s,
                          max_sequence=s, datatype_label=dt)
    w = eet.random_weights(cfg, vocab=8, seed=h + b).layers[0]
    x = np.random.default_rng(9).normal(0, 1, size=(b, s, h)).astype(np.float32)
    kv, acts = eet.preallocate_caches(cfg)
    if dt != "fp32":
        for t in kv._k + kv._v:
            t.fill_(float("nan"))
    out = eet.decoder_layer_forward(x.copy(), w, kv, desc, eet.Phase.PROMPT_PARALLEL, eet.BufferPool(), acts, 0)
    tol = 1e-5 if dt == "fp32" else 2e-2
    for i, n in enumerate(lengths):
        okv = orc.OracleKV(1, heads, n, h // heads, 1)
        ref = orc.decoder_layer(x[i:i + 1, :n], w, okv, (0,), 0, heads)
        assert np.isfinite(out[i, :n]).all(), f"row {i}: non-finite output"
        combined_close(out[i, :n], ref[0], tol, f"{dt} right-padded seq {i} (len {n})")


@pytest.mark.parametrize("dt", ["fp32", "bf16"])
def test_right_padded_encoder_layer(eet, dt):
    from oracle import eet_oracle as orc
    h, heads, lengths = 256, 4, [150, 37, 64, 100]
    desc = eet.make_batch(lengths, padding_side="right")
    s, b = desc.seq_len, len(lengths)
    cfg = eet.ModelConfig(batch_size=b, hidden_size=h, layer_count=1, head_count=heads, max_prompt=s,
                          max_sequence=s, datatype_label=dt)
    w = eet.random_weights(cfg, vocab=8, seed=5).layers[0]
    x = np.random.default_rng(10).normal(0, 1, size=(b, s, h)).astype(np.float32)
    out = eet.encoder_layer_forward(x.copy(), w, desc, eet.BufferPool(), head_count=heads, datatype_label=dt)
    tol = 1e-5 if dt == "fp32" else 2e-2
    for i, n in enumerate(lengths):
        ref = orc.encoder_layer(x[i:i + 1, :n], w, (0,), heads)
        combined_close(out[i, :n], ref[0], tol, f"{dt} right-padded encoder seq {i}")


def test_right_padding_matches_left_padding_bit_exact(eet):
    """The same sequences, right- vs left-padded: identical valid rows (the
    per-sequence work is the same; only the slot offsets differ)."""
    h, heads, lengths = 256, 4, [40, 17, 33]
    cfg = eet.ModelConfig(batch_size=3, hidden_size=h, layer_count=1, head_count=heads, max_prompt=40,
                          max_sequence=40)
    w = eet.random_weights(cfg, vocab=8, seed=3).layers[0]
    rows = [np.random.default_rng(i).normal(0, 1, size=(n, h)).astype(np.float32) for i, n in enumerate(lengths)]
    xr = np.zeros((3, 40, h), np.float32)
    xl = np.zeros((3, 40, h), np.float32)
    for i, (r, n) in enumerate(zip(rows, lengths)):
        xr[i, :n] = r
        xl[i, 40 - n:] = r
    kv, acts = eet.preallocate_caches(cfg)
    outr = eet.decoder_layer_forward(xr, w, kv, eet.make_batch(lengths, padding_side="right"),
                                     eet.Phase.PROMPT_PARALLEL, eet.BufferPool(), acts, 0)
    kv2, acts2 = eet.preallocate_caches(cfg)
    outl = eet.decoder_layer_forward(xl, w, kv2, eet.make_batch(lengths), eet.Phase.PROMPT_PARALLEL,
                                     eet.BufferPool(), acts2, 0)
    for i, n in enumerate(lengths):
        np.testing.assert_allclose(outr[i, :n], outl[i, 40 - n:], rtol=0, atol=1e-6)


def test_right_padded_incremental_step_rejected(eet):
    cfg = eet.ModelConfig(batch_size=2, hidden_size=64, layer_count=1, head_count=4, max_prompt=8, max_sequence=9)
    w = eet.random_weights(cfg, vocab=8, seed=1).layers[0]
    kv, acts = eet.preallocate_caches(cfg)
    desc = eet.make_batch([8, 5], padding_side="right")
    x = np.random.default_rng(0).normal(0, 1, size=(2, 8, 64)).astype(np.float32)
    eet.decoder_layer_forward(x, w, kv, desc, eet.Phase.PROMPT_PARALLEL, eet.BufferPool(), acts, 0)
    kv.advance(8)
    with pytest.raises(ValueError, match="left-padded"):
        eet.decoder_layer_forward(x[:, :1].copy(), w, kv, desc, eet.Phase.INCREMENTAL, eet.BufferPool(), acts, 0)
