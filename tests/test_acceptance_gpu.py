"""The reference's acceptance protocol (criteria 3 and 4,
/root/reference/pkg/tests/test_acceptance.py:126-204) restated against this
package on the GPU, plus NaN-poisoned variants for the 16-bit tensor-core
path.

* criterion 3: 100 seeded tiny models, ragged prompts, 1-8 greedy steps;
  fp32 tokens identical to the oracle (pinned to the reference's
  ``reference_generate`` goldens) and per-step logits within 1e-4.
* criterion 4: 100 decoder + 100 encoder cases; perturbed pad embeddings and
  poisoned pad-slot K/V (the reference's 77 / -77, and NaN) leave every
  valid output bit-identical.
* 16-bit: every K/V slot and every idle pool buffer filled with NaN before
  the prompt pass, at lengths whose valid window is not a multiple of the
  64-key attention tile and with seq == s_max; outputs must be finite and
  bit-identical to the clean (zero-initialised) run, for the decoder
  (prompt + incremental step) and the encoder.
"""

import numpy as np
import pytest
from numpy.testing import assert_allclose

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def eet(cuda_ok):
    import paper_2104_12470_b200 as m
    return m


def test_criterion_3_kv_cache_correctness_100_seeds(eet):
    from oracle import eet_oracle as orc
    cfg = eet.ModelConfig(batch_size=2, hidden_size=8, layer_count=2, head_count=2,
                          max_prompt=8, max_sequence=16)
    for seed in range(100):
        rng = np.random.default_rng(seed)
        w = eet.random_weights(cfg, vocab=16, seed=seed)
        prompts = [[int(t) for t in rng.integers(0, 16, size=rng.integers(1, 9))] for _ in range(2)]
        steps = int(rng.integers(1, 9))
        tr = eet.RunTrace(collect_logits=True)
        toks = eet.generate(w, eet.GenerationRequest(prompts=prompts, steps=steps), cfg, trace=tr)
        ref, logs = orc.generate(w, prompts, steps, 16, collect_logits=True)
        assert np.array_equal(toks, ref), f"seed {seed}"
        for ours, theirs in zip(tr.step_logits, logs):
            assert_allclose(ours, theirs, atol=1e-4)


@pytest.mark.parametrize("poison", [77.0, float("nan")])
def test_criterion_4_pad_invariance_100_cases(eet, poison):
    for case in range(100):
        rng = np.random.default_rng(1000 + case)
        batch = int(rng.integers(1, 4))
        seq = int(rng.integers(2, 9))
        pads = tuple(int(rng.integers(0, seq)) for _ in range(batch))
        desc = eet.BatchDescriptor(seq_len=seq, padding_len=pads, batch=batch)
        heads, hidden = 2, 8
        cfg = eet.ModelConfig(batch_size=batch, hidden_size=hidden, layer_count=1, head_count=heads,
                              max_prompt=seq, max_sequence=seq + 1)
        w = eet.random_weights(cfg, vocab=8, seed=case).layers[0]
        x = rng.normal(0, 1, (batch, seq, hidden)).astype(np.float32)
        x_pert = x.copy()
        for b in range(batch):
            x_pert[b, :pads[b]] = rng.normal(size=(pads[b], hidden)) if poison == 77.0 else np.nan
        step = np.random.default_rng(case).normal(0, 1, (batch, 1, hidden)).astype(np.float32)

        def decoder_run(inp, poisoned):
            kv, acts = eet.preallocate_caches(cfg)
            pool = eet.BufferPool()
            out = eet.decoder_layer_forward(inp.copy(), w, kv, desc, eet.Phase.PROMPT_PARALLEL, pool, acts, 0).copy()
            kv.advance(seq)
            if poisoned:
                for b in range(batch):
                    kv._k[0][b, :, :pads[b]] = poison
                    kv._v[0][b, :, :pads[b]] = -poison
            return out, eet.decoder_layer_forward(step.copy(), w, kv, desc, eet.Phase.INCREMENTAL, pool, acts, 0).copy()

        base, base_step = decoder_run(x, False)
        pert, pert_step = decoder_run(x_pert, True)
        for b in range(batch):
            assert np.array_equal(base[b, pads[b]:], pert[b, pads[b]:]), f"case {case} decoder"
        assert np.array_equal(base_step, pert_step), f"case {case} step"
        enc = eet.encoder_layer_forward(x.copy(), w, desc, eet.BufferPool(), head_count=heads)
        enc_p = eet.encoder_layer_forward(x_pert.copy(), w, desc, eet.BufferPool(), head_count=heads)
        for b in range(batch):
            assert np.array_equal(enc[b, pads[b]:], enc_p[b, pads[b]:]), f"case {case} encoder"


NAN_CASES = [
    # dt, h, heads, lengths, extra slots after the prompt
    ("bf16", 256, 4, [200, 77, 131], 0),        # hd 64, seq == s_max
    ("fp16", 256, 4, [200, 77, 131], 0),
    ("bf16", 512, 4, [190, 190, 1], 0),         # hd 128
    ("fp16", 512, 4, [300, 45], 3),             # room for incremental steps
    ("bf16", 1024, 16, [513, 100, 257, 64], 2),
]


@pytest.mark.parametrize("dt,h,heads,lengths,extra", NAN_CASES)
def test_nan_poisoned_cache_and_scratch_16bit(eet, dt, h, heads, lengths, extra):
    desc = eet.make_batch(lengths)
    s, b = desc.seq_len, len(lengths)
    assert any((s - p) % 64 for p in desc.padding_len)
    cfg = eet.ModelConfig(batch_size=b, hidden_size=h, layer_count=1, head_count=heads,
                          max_prompt=s, max_sequence=s + extra, datatype_label=dt)
    w = eet.random_weights(cfg, vocab=8, seed=h + b).layers[0]
    rng = np.random.default_rng(5)
    x = rng.normal(0, 1, size=(b, s, h)).astype(np.float32)
    steps = rng.normal(0, 1, size=(max(extra, 1), b, 1, h)).astype(np.float32)

    def run(poisoned):
        kv, acts = eet.preallocate_caches(cfg)
        pool = eet.BufferPool()
        inp = x.copy()
        if poisoned:
            for t in kv._k + kv._v:
                t.fill_(float("nan"))
            for i, pad in enumerate(desc.padding_len):
                inp[i, :pad] = np.nan
            # settle the pool's buffers, then poison every one of them
            kv0, acts0 = eet.preallocate_caches(cfg)
            eet.decoder_layer_forward(x.copy(), w, kv0, desc, eet.Phase.PROMPT_PARALLEL, pool, acts0, 0)
            pool.debug_fill(0xFF)
        out = eet.decoder_layer_forward(inp.copy(), w, kv, desc, eet.Phase.PROMPT_PARALLEL, pool, acts, 0)
        kv.advance(s)
        outs = [out]
        for j in range(extra):
            if poisoned:
                pool.debug_fill(0xFF)
            outs.append(eet.decoder_layer_forward(steps[j].copy(), w, kv, desc, eet.Phase.INCREMENTAL,
                                                  pool, acts, 0).copy())
            kv.advance(1)
        enc_pool = eet.BufferPool()
        if poisoned:
            eet.encoder_layer_forward(x.copy(), w, desc, enc_pool, head_count=heads, datatype_label=dt)
            enc_pool.debug_fill(0xFF)
        enc = eet.encoder_layer_forward(inp.copy(), w, desc, enc_pool, head_count=heads, datatype_label=dt)
        return outs, enc

    (clean, enc_clean), (dirty, enc_dirty) = run(False), run(True)
    for i, pad in enumerate(desc.padding_len):
        assert np.isfinite(dirty[0][i, pad:]).all(), f"{dt} prompt row {i} not finite"
        assert np.array_equal(clean[0][i, pad:], dirty[0][i, pad:]), f"{dt} prompt row {i}"
        assert np.isfinite(enc_dirty[i, pad:]).all(), f"{dt} encoder row {i} not finite"
        assert np.array_equal(enc_clean[i, pad:], enc_dirty[i, pad:]), f"{dt} encoder row {i}"
    for j in range(1, len(clean)):
        assert np.isfinite(dirty[j]).all() and np.array_equal(clean[j], dirty[j]), f"{dt} step {j}"
