"""Pin the CPU oracle to the golden vectors produced by the real reference.

These run on CPU (no GPU marker). The fixtures come from
``tests/golden/make_golden.py``, which imports the reference ``maskfold``.
"""

import hashlib

import numpy as np
import pytest
from numpy.testing import assert_allclose

from conftest import golden_meta, load_golden
from oracle import eet_oracle as orc


@pytest.fixture(scope="module")
def sm():
    return load_golden("softmax")


def test_causal_and_padding_softmax_match_reference(sm):
    for i in range(int(sm["n_cases"])):
        raw, pads, heads = sm[f"c{i}_raw"], tuple(sm[f"c{i}_pads"]), int(sm[f"c{i}_heads"])
        c = orc.masked_softmax(raw, pads, heads, causal=True)
        p = orc.masked_softmax(raw, pads, heads, causal=False)
        assert_allclose(c, sm[f"c{i}_causal"], atol=1e-6)
        assert_allclose(p, sm[f"c{i}_padding"], atol=1e-6)
        # exact zeros outside the window, as the reference writes them
        assert np.array_equal(c == 0, sm[f"c{i}_causal"] == 0)
        assert np.array_equal(p == 0, sm[f"c{i}_padding"] == 0)


def test_step_softmax_matches_reference(sm):
    for i in range(int(sm["n_step"])):
        out = orc.step_softmax(sm[f"s{i}_raw"], tuple(sm[f"s{i}_pads"]))
        assert_allclose(out, sm[f"s{i}_out"], atol=1e-6)


def test_folded_large_plane(sm):
    raw = np.random.default_rng(int(sm["big_seed"])).normal(0.0, 3.0, size=(1, 1030, 1030)).astype(np.float32)
    out = orc.masked_softmax(raw, tuple(sm["big_pads"]), 1, causal=True)[0, sm["big_rows"]]
    assert_allclose(out, sm["big_causal_rows"], atol=1e-6)


def test_mha_matches_reference():
    g = load_golden("mha")
    for i in range(int(g["n_cases"])):
        out = orc.mha(g[f"m{i}_q"], g[f"m{i}_k"], g[f"m{i}_v"], tuple(g[f"m{i}_pads"]),
                      int(g[f"m{i}_heads"]), causal=bool(g[f"m{i}_causal"]))
        assert_allclose(out, g[f"m{i}_out"], atol=1e-5)


def _digest(model):
    h = hashlib.sha256()
    arrays = [model.token_embedding, model.position_embedding]
    for lw in model.layers:
        arrays += [lw.ln1_scale, lw.ln1_shift, lw.wq, lw.wk, lw.wv, lw.wo,
                   lw.ln2_scale, lw.ln2_shift, lw.w1, lw.w2]
    arrays += [model.final_scale, model.final_shift, model.output_head]
    for a in arrays:
        h.update(np.ascontiguousarray(a, np.float32).tobytes())
    return h.hexdigest()


@pytest.mark.parametrize("name", ["tiny", "small", "hd64", "c1"])
def test_decoder_layer_matches_reference(name):
    g = load_golden("layers")
    m = golden_meta(g)[name]
    model = orc.seeded_weights(m["hidden"], 1, m["heads"], m["vocab"], m["max_sequence"], m["wseed"])
    assert _digest(model) == m["weights_sha256"], "seeded init drifted from the reference"
    w = model.layers[0]
    x = g[f"{name}_x"]
    pads = tuple(int(p) for p in g[f"{name}_pads"])
    b, h = m["batch"], m["hidden"]
    s = max(m["lengths"])
    kv = orc.OracleKV(b, m["heads"], m["max_sequence"], h // m["heads"], 1)
    out = orc.decoder_layer(x[:, :s], w, kv, pads, 0, m["heads"])
    ref = g[f"{name}_prompt_out"]
    for bi, pad in enumerate(pads):
        assert_allclose(out[bi, pad:], ref[bi, pad:], atol=2e-5, rtol=1e-5)
    kv.advance(s)
    steps = []
    for j in range(m["steps"]):
        steps.append(orc.decoder_layer(x[:, s + j:s + j + 1], w, kv, pads, 0, m["heads"]))
        kv.advance(1)
    if steps:
        assert_allclose(np.concatenate(steps, 1), g[f"{name}_step_out"], atol=2e-5, rtol=1e-5)
    enc = orc.encoder_layer(x[:, :s], w, pads, m["heads"])
    for bi, pad in enumerate(pads):
        assert_allclose(enc[bi, pad:], g[f"{name}_enc_out"][bi, pad:], atol=2e-5, rtol=1e-5)


def test_generate_matches_reference():
    g = load_golden("generate")
    meta = golden_meta(g)
    for key, m in meta.items():
        model = orc.seeded_weights(m["hidden"], m["layers"], m["heads"], m["vocab"],
                                   m["max_sequence"], m["seed"])
        assert _digest(model) == m["weights_sha256"]
        flat = g[f"{key}_prompts"]
        prompts = [[int(t) for t in row if t >= 0] for row in flat]
        toks, logs = orc.generate(model, prompts, m["steps"], m["max_sequence"], collect_logits=True)
        assert np.array_equal(toks, g[f"{key}_tokens"]), key
        assert_allclose(np.stack(logs), g[f"{key}_logits"], atol=1e-4)


def test_plumbing_vectors():
    g = load_golden("plumbing")
    assert orc.left_pads([5, 2, 4, 10]) == tuple(g["make_batch_5_2_4_10"])
    assert orc.lengths_for_ratio(4, 64, 0.2) == list(g["ratio_lengths_4_64_02"])
    assert orc.lengths_for_ratio(8, 512, 0.5) == list(g["ratio_lengths_8_512_05"])


def test_teacher_forcing_with_own_tokens_is_identity():
    """Forcing the reference's own tokens reproduces the free-running
    generate exactly (the forced mode only changes what is fed back)."""
    g = load_golden("generate")
    key, m = next(iter(golden_meta(g).items()))
    model = orc.seeded_weights(m["hidden"], m["layers"], m["heads"], m["vocab"], m["max_sequence"], m["seed"])
    prompts = [[int(t) for t in row if t >= 0] for row in g[f"{key}_prompts"]]
    toks, logs = orc.generate(model, prompts, m["steps"], m["max_sequence"], collect_logits=True)
    ft, flogs = orc.generate(model, prompts, m["steps"], m["max_sequence"], collect_logits=True, forced=toks)
    assert np.array_equal(ft, toks)
    assert all(np.array_equal(a, b) for a, b in zip(logs, flogs))
    # forcing other tokens changes later logits but step 0 stays put
    other = (toks + 1) % m["vocab"]
    _, olog = orc.generate(model, prompts, m["steps"], m["max_sequence"], collect_logits=True, forced=other)
    assert np.array_equal(olog[0], logs[0])


def test_layer_rows_equals_full_layer():
    """decoder_layer_rows (selected query slots) is bit-identical to the full
    prompt-phase layer on those slots, and writes the same K/V."""
    h, heads, s = 64, 4, 40
    model = orc.seeded_weights(h, 1, heads, 8, s + 1, 5)
    x = np.random.default_rng(1).normal(size=(3, s, h)).astype(np.float32)
    pads = (0, 9, 39)
    kv = orc.OracleKV(3, heads, s + 1, h // heads, 1)
    full = orc.decoder_layer(x, model.layers[0], kv, pads, 0, heads)
    rows = [0, 8, 9, 21, 39]
    kv2 = orc.OracleKV(3, heads, s + 1, h // heads, 1)
    part = orc.decoder_layer_rows(x, model.layers[0], pads, heads, rows, kv=kv2)
    for b, pad in enumerate(pads):
        for j, r in enumerate(rows):
            if r >= pad:
                assert np.array_equal(part[b, j], full[b, r])
    assert np.array_equal(kv.k[0], kv2.k[0]) and np.array_equal(kv.v[0], kv2.v[0])
