"""GPU parity of decoder_layer_forward / encoder_layer_forward / generate
against the reference's golden outputs (fp32 mode) and the CPU oracle
(16-bit modes), plus the reference's property tests (pad invariance,
poisoned cache slots, phase validation, allocation ledger)."""

import numpy as np
import pytest
from numpy.testing import assert_allclose

from conftest import combined_close, golden_meta, load_golden

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def eet(cuda_ok):
    import paper_2104_12470_b200 as m
    return m


def _cfg(eet, b, h, heads, p, s, layers=1, dt="fp32"):
    return eet.ModelConfig(batch_size=b, hidden_size=h, layer_count=layers, head_count=heads,
                           max_prompt=p, max_sequence=s, datatype_label=dt)


# ----------------------------------------------------------- fp32 goldens
@pytest.mark.parametrize("name", ["tiny", "small", "hd64", "c1"])
def test_decoder_layer_fp32_matches_reference(eet, name):
    """Prompt pass + incremental steps vs the reference's outputs on
    identical weights: north-star fp32 tolerance rtol 1e-5 (combined form,
    SURVEY Appendix B.3) on valid rows; K cache equal too."""
    g = load_golden("layers")
    m = golden_meta(g)[name]
    b, h, heads, steps = m["batch"], m["hidden"], m["heads"], m["steps"]
    s = max(m["lengths"])
    cfg = _cfg(eet, b, h, heads, s, m["max_sequence"])
    w = eet.random_weights(cfg, vocab=m["vocab"], seed=m["wseed"]).layers[0]
    desc = eet.make_batch(m["lengths"])
    x = g[f"{name}_x"]
    kv, acts = eet.preallocate_caches(cfg)
    pool = eet.BufferPool()
    out = eet.decoder_layer_forward(x[:, :s].copy(), w, kv, desc, eet.Phase.PROMPT_PARALLEL, pool, acts, 0)
    ref = g[f"{name}_prompt_out"]
    for i, pad in enumerate(desc.padding_len):
        combined_close(out[i, pad:], ref[i, pad:], 1e-5, f"{name} prompt row {i}")
    kv.advance(s)
    outs = []
    for j in range(steps):
        outs.append(eet.decoder_layer_forward(x[:, s + j:s + j + 1].copy(), w, kv, desc,
                                              eet.Phase.INCREMENTAL, pool, acts, 0).copy())
        kv.advance(1)
    if steps:
        combined_close(np.concatenate(outs, 1), g[f"{name}_step_out"], 1e-5, f"{name} steps")
    if h <= 128:
        kc = kv._k[0][:, :, :s + steps].cpu().numpy()
        refk = g[f"{name}_kcache"]
        for i, pad in enumerate(desc.padding_len):
            combined_close(kc[i, :, pad:], refk[i, :, pad:], 1e-5, f"{name} K cache")


@pytest.mark.parametrize("name", ["tiny", "small", "hd64", "c1"])
def test_encoder_layer_fp32_matches_reference(eet, name):
    g = load_golden("layers")
    m = golden_meta(g)[name]
    s = max(m["lengths"])
    cfg = _cfg(eet, m["batch"], m["hidden"], m["heads"], s, m["max_sequence"])
    w = eet.random_weights(cfg, vocab=m["vocab"], seed=m["wseed"]).layers[0]
    desc = eet.make_batch(m["lengths"])
    out = eet.encoder_layer_forward(g[f"{name}_x"][:, :s].copy(), w, desc, eet.BufferPool(),
                                    head_count=m["heads"])
    ref = g[f"{name}_enc_out"]
    for i, pad in enumerate(desc.padding_len):
        combined_close(out[i, pad:], ref[i, pad:], 1e-5, f"{name} encoder row {i}")


# ----------------------------------------------------- 16-bit vs oracle
@pytest.mark.parametrize("dt", ["bf16", "fp16"])
@pytest.mark.parametrize("b,h,heads,lengths", [(4, 768, 12, [64, 47, 47, 47]),
                                                (3, 1024, 8, [200, 17, 129]),
                                                (2, 2048, 16, [300, 1]),
                                                # > 148 attention work items: the
                                                # persistent CTAs loop over items
                                                (6, 1024, 16, [900, 700, 1, 513, 256, 880]),
                                                (4, 2048, 16, [640, 300, 129, 600])])
def test_decoder_layer_16bit_vs_oracle(eet, dt, b, h, heads, lengths):
    """North-star 16-bit tolerance 2e-2 (combined) vs the fp32 oracle on the
    same fp32 weights; exercises the tcgen05 GEMMs (T > 16 rows) and the
    decode path (GEMV + split-K attention)."""
    from oracle import eet_oracle as orc
    desc = eet.make_batch(lengths)
    s = desc.seq_len
    cfg = _cfg(eet, b, h, heads, s, s + 2, dt=dt)
    w = eet.random_weights(cfg, vocab=8, seed=7)
    x = np.random.default_rng(3).normal(0, 1, size=(b, s + 2, h)).astype(np.float32)
    kv, acts = eet.preallocate_caches(cfg)
    pool = eet.BufferPool()
    out = eet.decoder_layer_forward(x[:, :s].copy(), w.layers[0], kv, desc, eet.Phase.PROMPT_PARALLEL, pool, acts, 0)
    kv.advance(s)
    st = eet.decoder_layer_forward(x[:, s:s + 1].copy(), w.layers[0], kv, desc, eet.Phase.INCREMENTAL, pool, acts, 0)
    om = orc.seeded_weights(h, 1, heads, 8, s + 2, 7)
    okv = orc.OracleKV(b, heads, s + 2, h // heads, 1)
    ref = orc.decoder_layer(x[:, :s], om.layers[0], okv, desc.padding_len, 0, heads)
    okv.advance(s)
    ref_st = orc.decoder_layer(x[:, s:s + 1], om.layers[0], okv, desc.padding_len, 0, heads)
    for i, pad in enumerate(desc.padding_len):
        combined_close(out[i, pad:], ref[i, pad:], 2e-2, f"{dt} prompt row {i}")
    combined_close(st, ref_st, 2e-2, f"{dt} step")


# ------------------------------------------------------------ properties
def _layer(eet, cfg, seed):
    return eet.random_weights(cfg, vocab=8, seed=seed).layers[0]


def test_zero_weights_identity(eet):
    cfg = _cfg(eet, 2, 8, 2, 4, 4)
    kv, acts = eet.preallocate_caches(cfg)
    z = lambda *s: np.zeros(s, np.float32)  # noqa: E731
    w = eet.LayerWeights(z(8), z(8), z(8, 8), z(8, 8), z(8, 8), z(8, 8), z(8), z(8), z(8, 32), z(32, 8))
    x = np.random.default_rng(0).normal(0, 1, size=(2, 4, 8)).astype(np.float32)
    out = eet.decoder_layer_forward(x.copy(), w, kv, eet.make_batch([4, 3]), eet.Phase.PROMPT_PARALLEL,
                                    eet.BufferPool(), acts, 0)
    assert np.array_equal(out, x)


def test_pad_slot_perturbation_invisible(eet):
    """Bit-exact: pad rows are never read (test_runtime.py:122-143)."""
    cfg = _cfg(eet, 2, 8, 2, 6, 6)
    w = _layer(eet, cfg, 1)
    desc = eet.BatchDescriptor(seq_len=6, padding_len=(3, 1), batch=2)
    rng = np.random.default_rng(8)
    x = rng.normal(0, 1, size=(2, 6, 8)).astype(np.float32)
    x2 = x.copy()
    for b, pad in enumerate(desc.padding_len):
        x2[b, :pad] = rng.normal(size=(pad, 8))
    outs = []
    for inp in (x, x2):
        kv, acts = eet.preallocate_caches(cfg)
        outs.append(eet.decoder_layer_forward(inp.copy(), w, kv, desc, eet.Phase.PROMPT_PARALLEL,
                                              eet.BufferPool(), acts, 0))
    for b, pad in enumerate(desc.padding_len):
        assert np.array_equal(outs[0][b, pad:], outs[1][b, pad:])


@pytest.mark.parametrize("dt", ["fp32", "bf16"])
def test_cached_pad_slots_never_read(eet, dt):
    """Poisoned K/V at pad slots must not change a later step, bit-exact
    (test_runtime.py:145-172, acceptance criterion 4)."""
    h = 8 if dt == "fp32" else 64
    cfg = _cfg(eet, 2, h, 2, 4, 6, dt=dt)
    w = _layer(eet, cfg, 4)
    desc = eet.BatchDescriptor(seq_len=4, padding_len=(2, 0), batch=2)
    rng = np.random.default_rng(3)
    x = rng.normal(0, 1, size=(2, 4, h)).astype(np.float32)
    step = rng.normal(0, 1, size=(2, 1, h)).astype(np.float32)

    def run(poison):
        kv, acts = eet.preallocate_caches(cfg)
        pool = eet.BufferPool()
        eet.decoder_layer_forward(x.copy(), w, kv, desc, eet.Phase.PROMPT_PARALLEL, pool, acts, 0)
        kv.advance(4)
        if poison:
            kv._k[0][0, :, :2] = 99.0
            kv._v[0][0, :, :2] = -99.0
        return eet.decoder_layer_forward(step.copy(), w, kv, desc, eet.Phase.INCREMENTAL, pool, acts, 0)

    assert np.array_equal(run(False), run(True))


def test_uneven_batch_matches_single_runs(eet):
    cfg = _cfg(eet, 4, 8, 2, 10, 10)
    w = _layer(eet, cfg, 9)
    lengths = [5, 2, 4, 10]
    desc = eet.make_batch(lengths)
    x = np.random.default_rng(2).normal(0, 1, size=(4, 10, 8)).astype(np.float32)
    kv, acts = eet.preallocate_caches(cfg)
    batched = eet.decoder_layer_forward(x.copy(), w, kv, desc, eet.Phase.PROMPT_PARALLEL, eet.BufferPool(), acts, 0)
    for i, n in enumerate(lengths):
        cfg1 = _cfg(eet, 1, 8, 2, n, n)
        kv1, acts1 = eet.preallocate_caches(cfg1)
        pad = desc.padding_len[i]
        alone = eet.decoder_layer_forward(x[i:i + 1, pad:].copy(), w, kv1, eet.make_batch([n]),
                                          eet.Phase.PROMPT_PARALLEL, eet.BufferPool(), acts1, 0)
        assert_allclose(batched[i, pad:], alone[0], atol=1e-5)


def test_phase_validation(eet):
    cfg = _cfg(eet, 1, 8, 2, 4, 4)
    w = _layer(eet, cfg, 0)
    kv, acts = eet.preallocate_caches(cfg)
    desc = eet.make_batch([4])
    x = np.zeros((1, 4, 8), np.float32)
    with pytest.raises(ValueError, match="incremental step"):
        eet.decoder_layer_forward(x, w, kv, desc, eet.Phase.INCREMENTAL, eet.BufferPool(), acts, 0)
    with pytest.raises(ValueError, match="before the prompt"):
        eet.decoder_layer_forward(x[:, :1], w, kv, desc, eet.Phase.INCREMENTAL, eet.BufferPool(), acts, 0)
    kv.advance(4)
    with pytest.raises(ValueError, match="empty cache"):
        eet.decoder_layer_forward(x, w, kv, desc, eet.Phase.PROMPT_PARALLEL, eet.BufferPool(), acts, 0)


def test_cuda_tensor_inputs_in_place(eet):
    """CUDA tensors (incl. the strided acts.hidden view) are updated in place."""
    cfg = _cfg(eet, 2, 64, 4, 8, 8)
    w = _layer(eet, cfg, 2)
    desc = eet.make_batch([6, 4])
    kv, acts = eet.preallocate_caches(cfg)
    xs = torch.randn(2, 6, 64)
    acts.hidden[:2, :6] = xs.cuda()
    view = acts.hidden[:2, :6]
    kv2, acts2 = eet.preallocate_caches(cfg)
    host = eet.decoder_layer_forward(xs.numpy().copy(), w, kv2, desc, eet.Phase.PROMPT_PARALLEL,
                                     eet.BufferPool(), acts2, 0)
    out = eet.decoder_layer_forward(view, w, kv, desc, eet.Phase.PROMPT_PARALLEL, eet.BufferPool(), acts, 0)
    assert out is view
    got = acts.hidden[:2, :6].cpu().numpy()
    for i, pad in enumerate(desc.padding_len):
        assert np.array_equal(got[i, pad:], host[i, pad:])


def test_layer_requests_scratch_from_the_pool(eet):
    """No mask tensor and no score tensor: the fused path's pool requests are
    the linear activation buffers only (test_runtime.py:300-314)."""
    cfg = _cfg(eet, 2, 16, 2, 8, 12)
    w = _layer(eet, cfg, 0)
    log = eet.AllocationLog()
    pool = eet.BufferPool(log=log)
    kv, acts = eet.preallocate_caches(cfg, log=log)
    desc = eet.make_batch([8, 8])
    x = np.random.default_rng(0).normal(size=(2, 8, 16)).astype(np.float32)
    eet.decoder_layer_forward(x, w, kv, desc, eet.Phase.PROMPT_PARALLEL, pool, acts, 0)
    kv.advance(8)
    after_prompt = len(log.records)
    for _ in range(3):
        eet.decoder_layer_forward(x[:, :1].copy(), w, kv, desc, eet.Phase.INCREMENTAL, pool, acts, 0)
        kv.advance(1)
    tags = {r.tag for r in log.records if r.event == "request"}
    assert tags == {"attention.layernorm", "attention.query", "attention.context",
                    "ffn.layernorm", "ffn.intermediate"}
    assert all("mask" not in r.tag and "scores" not in r.tag for r in log.records)
    linear_cap = 2 * 8 * 4 * 16
    assert all(r.size <= linear_cap for r in log.records if r.event == "request")
    # decode steps reuse the prompt's buffers: no malloc after the prompt pass
    assert all(r.decision != "malloc" for r in log.records[after_prompt:])


# -------------------------------------------------------------- generate
def test_generate_fp32_matches_reference(eet):
    """Greedy tokens identical and logits within 1e-4 of the reference on
    every golden seed (acceptance criterion 3)."""
    g = load_golden("generate")
    for key, m in golden_meta(g).items():
        cfg = _cfg(eet, m["batch"], m["hidden"], m["heads"], m["max_prompt"], m["max_sequence"], m["layers"])
        w = eet.random_weights(cfg, m["vocab"], m["seed"])
        prompts = [[int(t) for t in row if t >= 0] for row in g[f"{key}_prompts"]]
        tr = eet.RunTrace(collect_logits=True)
        toks = eet.generate(w, eet.GenerationRequest(prompts=prompts, steps=m["steps"]), cfg, trace=tr)
        assert np.array_equal(toks, g[f"{key}_tokens"]), key
        assert_allclose(np.stack(tr.step_logits), g[f"{key}_logits"], atol=1e-4)


def test_generate_graph_equals_eager(eet):
    cfg = _cfg(eet, 3, 64, 4, 12, 24, 2)
    w = eet.random_weights(cfg, 64, 5)
    req = eet.GenerationRequest(prompts=[[1, 2, 3], [4, 5, 6, 7, 8, 9], [10]], steps=10)
    a = eet.generate(w, req, cfg, use_graph=True)
    b = eet.generate(w, req, cfg, use_graph=False)
    assert np.array_equal(a, b)
    assert np.array_equal(a, eet.generate(w, req, cfg))


def test_generate_semantics(eet):
    cfg = _cfg(eet, 3, 8, 2, 8, 16, 2)
    w = eet.random_weights(cfg, 16, 0)
    kv, acts = eet.preallocate_caches(cfg)
    toks = eet.generate(w, eet.GenerationRequest(prompts=[[1, 2, 3], [4, 5, 6, 7], [8]], steps=0), cfg,
                        caches=(kv, acts))
    assert toks.shape == (3, 0) and kv.filled == 4
    same = eet.generate(w, eet.GenerationRequest(prompts=[[3, 1, 2]] * 3, steps=5), cfg)
    assert np.array_equal(same[0], same[1]) and np.array_equal(same[0], same[2])
    tr = eet.RunTrace()
    eet.generate(w, eet.GenerationRequest(prompts=[[1, 2, 3, 4]] * 2, steps=5), cfg, trace=tr)
    assert (tr.prompt_passes, tr.decode_steps, tr.layer_invocations) == (1, 5, 12)
    log = eet.AllocationLog()
    eet.generate(w, eet.GenerationRequest(prompts=[[1, 2, 3], [4, 5, 6]], steps=8), cfg, log=log)
    cache = [r for r in log.records if r.tag in ("kv_cache", "activation")]
    assert len(cache) == 2 and all(r.event == "preallocate" for r in cache)
    for req, frag in [(eet.GenerationRequest(prompts=[[1] * 8], steps=9), "max sequence"),
                      (eet.GenerationRequest(prompts=[[1] * 9], steps=0), "max prompt"),
                      (eet.GenerationRequest(prompts=[[1]] * 4, steps=0), "batch"),
                      (eet.GenerationRequest(prompts=[[16]], steps=0), "vocab")]:
        with pytest.raises(ValueError, match=frag):
            eet.generate(w, req, cfg)
    kv, acts = eet.preallocate_caches(cfg)
    kv.advance(1)
    with pytest.raises(ValueError, match="not empty"):
        eet.generate(w, eet.GenerationRequest(prompts=[[1, 2]], steps=0), cfg, caches=(kv, acts))


@pytest.mark.parametrize("dt", ["bf16", "fp16"])
def test_generate_16bit_first_logits_vs_oracle(eet, dt):
    """16-bit generate: the first step's logits (prompt pass + head) within
    2e-2 of the fp32 oracle; later tokens may legitimately diverge."""
    from oracle import eet_oracle as orc
    cfg = _cfg(eet, 2, 256, 4, 20, 32, 2, dt=dt)
    w = eet.random_weights(cfg, 128, 1)
    prompts = [list(range(1, 21)), [5, 6, 7]]
    tr = eet.RunTrace(collect_logits=True)
    eet.generate(w, eet.GenerationRequest(prompts=prompts, steps=3), cfg, trace=tr)
    _, logs = orc.generate(orc.seeded_weights(256, 2, 4, 128, 32, 1), prompts, 3, 32, collect_logits=True)
    combined_close(tr.step_logits[0], logs[0], 2e-2, f"{dt} first logits")


# --------------------------------------------------------- tensor parallel
@pytest.mark.parametrize("dt,h,heads,tp,lengths", [("fp32", 256, 8, 2, [40, 17]),
                                                   ("bf16", 1024, 8, 2, [300, 129]),
                                                   ("bf16", 1536, 12, 4, [256])])
def test_tensor_parallel_shards_sum_to_full_layer(eet, dt, h, heads, tp, lengths):
    """tp ranks emulated on one GPU: every rank's attention / FFN partial
    through the C ABI, summed (the all-reduce), residual-added — prompt pass
    and one decode step — equal the unsharded oracle layer."""
    from oracle import eet_oracle as orc
    from paper_2104_12470_b200 import _lib
    from paper_2104_12470_b200.tp import TensorParallelLayer, shard_config
    desc = eet.make_batch(lengths)
    s, b = desc.seq_len, len(lengths)
    cfg = _cfg(eet, b, h, heads, s, s + 1, dt=dt)
    w = eet.random_weights(cfg, vocab=8, seed=21).layers[0]
    xh = np.random.default_rng(4).normal(0, 1, size=(b, s + 1, h)).astype(np.float32)
    pool = eet.BufferPool()
    ranks = [TensorParallelLayer(w, cfg, r, tp, pool) for r in range(tp)]
    caches = [eet.preallocate_caches(shard_config(cfg, tp))[0] for _ in range(tp)]
    x = torch.from_numpy(xh[:, :s].copy()).cuda()

    def layer(x, phase):
        parts = [rk.attention_partial(x, kv, desc, phase, 0) for rk, kv in zip(ranks, caches)]
        total = torch.stack(parts).sum(0)
        ranks[0].residual_add(x, total)
        for rk in ranks:
            rk._rows = total.shape[0]
        ff = torch.stack([rk.ffn_partial(x) for rk in ranks]).sum(0)
        ranks[0].residual_add(x, ff)

    layer(x, _lib.PHASE_PROMPT)
    for kv in caches:
        kv.advance(s)
    x1 = torch.from_numpy(xh[:, s:].copy()).cuda()
    layer(x1, _lib.PHASE_INCREMENTAL)
    om = orc.seeded_weights(h, 1, heads, 8, s + 1, 21)
    okv = orc.OracleKV(b, heads, s + 1, h // heads, 1)
    ref = orc.decoder_layer(xh[:, :s], om.layers[0], okv, desc.padding_len, 0, heads)
    okv.advance(s)
    ref1 = orc.decoder_layer(xh[:, s:], om.layers[0], okv, desc.padding_len, 0, heads)
    tol = 1e-5 if dt == "fp32" else 2e-2
    got = x.cpu().numpy()
    for i, pad in enumerate(desc.padding_len):
        combined_close(got[i, pad:], ref[i, pad:], tol, f"tp{tp} prompt row {i}")
    combined_close(x1.cpu().numpy(), ref1, tol, f"tp{tp} decode step")



def test_ffn_chunked_reference_memory_shape(cuda_ok):
    """EET_FFN_CHUNKED=1 (fp32): the FFN intermediate is accumulated in two
    half-width chunks like the reference (runtime.py:195-214): no pool
    request wider than T x 2h, oracle parity at 1e-5, and the same greedy
    tokens as the default whole-width path (this process)."""
    import os
    import subprocess
    import sys
    import paper_2104_12470_b200 as eet
    code = r'''
import numpy as np, paper_2104_12470_b200 as eet
from oracle import eet_oracle as orc
cfg = eet.ModelConfig(batch_size=2, hidden_size=256, layer_count=2, head_count=4, max_prompt=40, max_sequence=48)
w = eet.random_weights(cfg, vocab=64, seed=4)
desc = eet.make_batch([40, 23])
x = np.random.default_rng(1).normal(0, 1, size=(2, 40, 256)).astype(np.float32)
kv, acts = eet.preallocate_caches(cfg)
log = eet.AllocationLog()
out = eet.decoder_layer_forward(x.copy(), w.layers[0], kv, desc, eet.Phase.PROMPT_PARALLEL,
                                eet.BufferPool(log=log), acts, 0)
okv = orc.OracleKV(2, 4, 40, 64, 1)
ref = orc.decoder_layer(x, w.layers[0], okv, desc.padding_len, 0, 4)
for i, p in enumerate(desc.padding_len):
    err = np.abs(out[i, p:] - ref[i, p:]).max() / (1 + np.abs(ref[i, p:]).max())
    assert err < 1e-5, err
T = sum(40 - p for p in desc.padding_len)
mids = [r.size for r in log.records if r.event == "request" and r.tag == "ffn.intermediate"]
assert mids and max(mids) <= T * 2 * 256, mids
req = eet.GenerationRequest(prompts=[[1, 2, 3, 4, 5], [7, 8]], steps=6)
print("TOKENS", eet.generate(w, req, cfg).tolist())
'''
    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, EET_FFN_CHUNKED="1", PYTHONPATH=repo)
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    toks = [l for l in r.stdout.splitlines() if l.startswith("TOKENS")][0]
    cfg = eet.ModelConfig(batch_size=2, hidden_size=256, layer_count=2, head_count=4, max_prompt=40,
                          max_sequence=48)
    w = eet.random_weights(cfg, vocab=64, seed=4)
    req = eet.GenerationRequest(prompts=[[1, 2, 3, 4, 5], [7, 8]], steps=6)
    assert toks == "TOKENS " + str(eet.generate(w, req, cfg).tolist())
