#!/usr/bin/env python3
"""Generate the golden parity vectors from the REAL reference implementation.

Runs only in the build container, where the reference ``maskfold`` package is
importable from ``/root/reference/pkg/src`` (read-only; it never travels to
the GPU box). The outputs are small ``.npz`` fixtures committed next to this
script; tests load them without touching ``/root/reference``.

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

Every fixture records what produced it (reference call + seed) in its keys.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

REF_SRC = os.environ.get("MASKFOLD_SRC", "/root/reference/pkg/src")
sys.path.insert(0, REF_SRC)
sys.dont_write_bytecode = True

import maskfold as mf  # noqa: E402
from maskfold import reference as mref  # noqa: E402
from maskfold.bench import prompt_lengths_for_ratio  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def rand_desc(rng, max_batch=4, max_seq=16):
    # same distribution as the reference tests' random_descriptor (conftest.py:68-73)
    batch = int(rng.integers(1, max_batch + 1))
    seq = int(rng.integers(1, max_seq + 1))
    pads = tuple(int(rng.integers(0, seq)) for _ in range(batch))
    return mf.BatchDescriptor(seq_len=seq, padding_len=pads, batch=batch)


def softmax_cases():
    rng = np.random.default_rng(2024)
    d = {}
    n = 300
    for i in range(n):
        desc = rand_desc(rng)
        heads = int(rng.integers(1, 5))
        raw = rng.normal(0.0, 3.0, size=(desc.batch * heads, desc.seq_len, desc.seq_len)).astype(np.float32)
        caus = mf.fused_causal_softmax(mf.AttentionScores(raw.copy(), desc.batch, heads), desc).data
        bidi = mf.fused_padding_softmax(mf.AttentionScores(raw.copy(), desc.batch, heads), desc).data
        d[f"c{i}_raw"] = raw
        d[f"c{i}_pads"] = np.asarray(desc.padding_len, np.int32)
        d[f"c{i}_heads"] = np.int32(heads)
        d[f"c{i}_causal"] = caus
        d[f"c{i}_padding"] = bidi
    # step softmax
    for i in range(100):
        L = int(rng.integers(1, 40))
        b = int(rng.integers(1, 5))
        heads = int(rng.integers(1, 5))
        pads = tuple(int(rng.integers(0, L)) for _ in range(b))
        desc = mf.BatchDescriptor(seq_len=L, padding_len=pads, batch=b)
        raw = rng.normal(0.0, 3.0, size=(b, heads, L)).astype(np.float32)
        d[f"s{i}_raw"] = raw
        d[f"s{i}_pads"] = np.asarray(pads, np.int32)
        d[f"s{i}_out"] = mf.fused_step_softmax(raw.copy(), desc)
    # a folded (multi-sub-block) causal plane: s = 1030 -> plan (2, 515)
    # (the raw plane is regenerated from its seed; only sampled rows are stored)
    desc = mf.BatchDescriptor(seq_len=1030, padding_len=(7,), batch=1)
    raw = np.random.default_rng(555).normal(0.0, 3.0, size=(1, 1030, 1030)).astype(np.float32)
    rows = np.asarray([0, 6, 7, 8, 100, 514, 515, 516, 1000, 1029])
    d["big_seed"] = np.int32(555)
    d["big_pads"] = np.asarray(desc.padding_len, np.int32)
    d["big_rows"] = rows
    d["big_causal_rows"] = mf.fused_causal_softmax(mf.AttentionScores(raw.copy(), 1, 1), desc).data[0, rows]
    d["n_cases"] = np.int32(n)
    d["n_step"] = np.int32(100)
    np.savez_compressed(os.path.join(OUT, "softmax.npz"), **d)


def mha_cases():
    rng = np.random.default_rng(7)
    d = {}
    n = 60
    for i in range(n):
        desc = rand_desc(rng, max_batch=3, max_seq=24)
        heads = int(rng.choice([1, 2, 4]))
        hd = int(rng.choice([4, 8, 16, 32, 64]))
        h = heads * hd
        q, k, v = (rng.normal(0, 1, size=(desc.batch, desc.seq_len, h)).astype(np.float32) for _ in range(3))
        causal = bool(i % 2 == 0)
        d[f"m{i}_q"], d[f"m{i}_k"], d[f"m{i}_v"] = q, k, v
        d[f"m{i}_pads"] = np.asarray(desc.padding_len, np.int32)
        d[f"m{i}_heads"] = np.int32(heads)
        d[f"m{i}_causal"] = np.int32(causal)
        d[f"m{i}_out"] = mf.mha_forward(q, k, v, desc, heads, causal=causal)
    d["n_cases"] = np.int32(n)
    np.savez_compressed(os.path.join(OUT, "mha.npz"), **d)


def weights_digest(w):
    hsh = hashlib.sha256()
    for a in w.arrays():
        hsh.update(np.ascontiguousarray(a, np.float32).tobytes())
    return hsh.hexdigest()


def layer_cases():
    """decoder_layer_forward prompt pass + incremental steps on several shapes."""
    d = {}
    specs = [
        # name, batch, hidden, heads, lengths, steps, wseed, xseed
        ("tiny", 2, 8, 2, [5, 3], 4, 3, 5),
        ("small", 3, 64, 4, [12, 5, 9], 5, 11, 12),
        ("hd64", 2, 128, 2, [33, 20], 3, 4, 6),
        # c1 shape: h=768, 12 heads, b=4, s=64; the bench's right-padded
        # lengths [64,47,47,47] are laid out in the reference's left-pad form
        ("c1", 4, 768, 12, prompt_lengths_for_ratio(4, 64, 0.2), 2, 0, 1),
    ]
    meta = {}
    for name, b, h, heads, lengths, steps, wseed, xseed in specs:
        desc = mf.make_batch(lengths)
        s = desc.seq_len
        cfg = mf.ModelConfig(batch_size=b, hidden_size=h, layer_count=1, head_count=heads,
                             max_prompt=s, max_sequence=s + steps)
        w = mf.random_weights(cfg, vocab=8, seed=wseed)
        lw = w.layers[0]
        rng = np.random.default_rng(xseed)
        x = rng.normal(0, 1, size=(b, s + steps, h)).astype(np.float32)
        kv, acts = mf.preallocate_caches(cfg)
        pool = mf.BufferPool()
        out = mf.decoder_layer_forward(x[:, :s].copy(), lw, kv, desc, mf.Phase.PROMPT_PARALLEL,
                                       pool, acts, 0).copy()
        kv.advance(s)
        step_outs = []
        for m in range(steps):
            xm = x[:, s + m:s + m + 1].copy()
            step_outs.append(mf.decoder_layer_forward(xm, lw, kv, desc, mf.Phase.INCREMENTAL,
                                                      pool, acts, 0).copy())
            kv.advance(1)
        d[f"{name}_x"] = x
        d[f"{name}_pads"] = np.asarray(desc.padding_len, np.int32)
        d[f"{name}_prompt_out"] = out
        d[f"{name}_step_out"] = np.concatenate(step_outs, axis=1) if steps else np.zeros((b, 0, h), np.float32)
        d[f"{name}_kcache"] = kv._k[0][:, :, :s + steps].copy() if h <= 128 else np.zeros(1, np.float32)
        # encoder layer on the same prompt input (bidirectional, runtime.py:266-301)
        d[f"{name}_enc_out"] = mf.encoder_layer_forward(x[:, :s].copy(), lw, desc, mf.BufferPool(),
                                                        head_count=heads).copy()
        meta[name] = dict(batch=b, hidden=h, heads=heads, lengths=list(lengths), steps=steps,
                          wseed=wseed, xseed=xseed, vocab=8, max_sequence=s + steps,
                          weights_sha256=weights_digest(w))
    d["meta"] = np.frombuffer(json.dumps(meta).encode(), dtype=np.uint8)
    np.savez_compressed(os.path.join(OUT, "layers.npz"), **d)


def generate_cases():
    d = {}
    meta = {}
    specs = [
        # name, batch, hidden, layers, heads, max_prompt, max_seq, vocab, n_seeds
        ("tiny", 3, 8, 2, 2, 8, 16, 16, 12),
        ("mid", 4, 64, 2, 4, 12, 24, 64, 4),
        ("wide", 2, 256, 2, 4, 20, 32, 128, 2),
    ]
    for name, b, h, nl, heads, p, smax, vocab, nseeds in specs:
        cfg = mf.ModelConfig(batch_size=b, hidden_size=h, layer_count=nl, head_count=heads,
                             max_prompt=p, max_sequence=smax)
        for seed in range(nseeds):
            rng = np.random.default_rng(100 + seed)
            w = mf.random_weights(cfg, vocab=vocab, seed=seed)
            prompts = [[int(t) for t in rng.integers(0, vocab, size=rng.integers(1, p + 1))]
                       for _ in range(int(rng.integers(1, b + 1)))]
            steps = int(rng.integers(1, smax - max(len(q) for q in prompts) + 1))
            steps = min(steps, 10)
            req = mf.GenerationRequest(prompts=prompts, steps=steps)
            tr = mf.RunTrace(collect_logits=True)
            toks = mf.generate(w, req, cfg, trace=tr)
            ref = mref.reference_generate(w, req, cfg)
            assert np.array_equal(toks, ref)
            key = f"{name}_{seed}"
            d[f"{key}_tokens"] = toks
            d[f"{key}_logits"] = np.stack(tr.step_logits)
            flat = np.full((len(prompts), p), -1, np.int64)
            for i, q in enumerate(prompts):
                flat[i, :len(q)] = q
            d[f"{key}_prompts"] = flat
            meta[key] = dict(batch=b, hidden=h, layers=nl, heads=heads, max_prompt=p,
                             max_sequence=smax, vocab=vocab, seed=seed, steps=steps,
                             weights_sha256=weights_digest(w))
    d["meta"] = np.frombuffer(json.dumps(meta).encode(), dtype=np.uint8)
    np.savez_compressed(os.path.join(OUT, "generate.npz"), **d)


def plumbing_cases():
    """Host-side plumbing: folding plans, make_batch, pool decision traces."""
    d = {}
    sizes = list(range(1, 70)) + [1023, 1024, 1025, 1030, 1280, 2048, 3000, 4096, 12288, 16384]
    caps = [1024, 4, 3, 100]
    rows = []
    for cap in caps:
        for sz in sizes:
            p = mf.plan_folding(sz, unit_cap=cap)
            rows.append((sz, cap, p.fold_count, p.sub_block_count, p.threads_per_block))
    d["fold"] = np.asarray(rows, np.int64)
    rng = np.random.default_rng(99)
    # pool traces: (size, scope, release) -> (capacity, decision)
    traces = []
    for _ in range(40):
        pool = mf.BufferPool()
        live = []
        for _ in range(int(rng.integers(5, 40))):
            size = int(rng.integers(1, 60))
            scope = "within" if rng.random() < 0.5 else "across"
            h = pool.request(size, scope=scope, tag="t")
            dec = pool.log.records[-1].decision
            # (step, size, within?, granted capacity, reused?, buffer index)
            traces.append((len(traces), size, scope == "within", h.capacity, dec == "reuse", h._index))
            live.append(h)
            if rng.random() < 0.6:
                victim = live.pop(int(rng.integers(0, len(live))))
                victim.release()
                traces.append((len(traces), -1, 0, victim.capacity, 0, victim._index))
        traces.append((len(traces), 0, 0, 0, 0, 0))   # trace separator
        traces.append((len(traces), pool.stats()["total_capacity"], pool.stats()["peak_in_use"],
                       pool.stats()["malloc_count"], pool.stats()["reuse_count"], 0))
    d["pool_traces"] = np.asarray(traces, np.int64)
    mb = mf.make_batch([5, 2, 4, 10])
    d["make_batch_5_2_4_10"] = np.asarray(mb.padding_len, np.int64)
    d["ratio_lengths_4_64_02"] = np.asarray(prompt_lengths_for_ratio(4, 64, 0.2), np.int64)
    d["ratio_lengths_8_512_05"] = np.asarray(prompt_lengths_for_ratio(8, 512, 0.5), np.int64)
    np.savez_compressed(os.path.join(OUT, "plumbing.npz"), **d)


def main():
    softmax_cases()
    mha_cases()
    layer_cases()
    generate_cases()
    plumbing_cases()
    for f in sorted(os.listdir(OUT)):
        if f.endswith(".npz"):
            print(f, os.path.getsize(os.path.join(OUT, f)))


if __name__ == "__main__":
    main()
