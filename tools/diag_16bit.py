#!/usr/bin/env python3
"""16-bit error budget: our kernels vs a torch emulation of the same
roundings (weights, GEMM inputs, q/k/v, P, ctx, mid in the 16-bit type; fp32
accumulation and residual stream), both against the fp32 oracle. If the two
errors are of the same size, a tolerance miss is the format's, not a bug."""
import math, os, sys
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2104_12470_b200 as eet  # noqa: E402
from oracle import eet_oracle as orc  # noqa: E402

torch.backends.cuda.matmul.allow_tf32 = False


def emu_layer(x, w, pads, heads, td):
    """x [b, t, h] fp32 cuda; prompt phase, causal, left pads."""
    b, t, h = x.shape
    hd = h // heads
    W = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda().to(td)  # noqa: E731
    def ln(v, g, bb):
        return torch.nn.functional.layer_norm(v, (h,), torch.from_numpy(g).cuda(), torch.from_numpy(bb).cuda(), 1e-5)
    l1 = ln(x, w.ln1_scale, w.ln1_shift).to(td)
    q, k, v = (l1 @ W(w.wq)), (l1 @ W(w.wk)), (l1 @ W(w.wv))
    sp = lambda a: a.view(b, t, heads, hd).transpose(1, 2)  # noqa: E731
    s = (sp(q).float() @ sp(k).float().transpose(2, 3)) * (1.0 / math.sqrt(hd))
    i = torch.arange(t, device="cuda")
    mask = (i[None, :] <= i[:, None])[None, None] & (i[None, None, None, :] >= torch.tensor(pads, device="cuda")[:, None, None, None])
    s = s.masked_fill(~mask, float("-inf"))
    p = torch.softmax(s, -1).nan_to_num(0.0).to(td)
    ctx = (p @ sp(v)).transpose(1, 2).reshape(b, t, h).to(td)
    x = x + (ctx @ W(w.wo)).float()
    l2 = ln(x, w.ln2_scale, w.ln2_shift).to(td)
    mid = l2 @ W(w.w1)
    mid = (mid.float() * 0.5 * (1 + torch.tanh(math.sqrt(2 / math.pi) * (mid.float() + 0.044715 * mid.float() ** 3)))).to(td)
    return x + (mid @ W(w.w2)).float()


def stats(ours, ref, what):
    ours, ref = np.asarray(ours, np.float64), np.asarray(ref, np.float64)
    rms = np.sqrt(np.mean(ref * ref))
    err = np.abs(ours - ref)
    ratio = err / (2e-2 * np.abs(ref) + 2e-2 * rms)
    print(f"  {what:28s} rms err/rms ref {np.sqrt(np.mean(err**2))/rms:.4f}  max err/bound {ratio.max():.3f}  "
          f"n>1 {int((ratio > 1).sum())}", flush=True)


def gpt2m():
    cfg = eet.ModelConfig(1, 1024, 24, 16, 512, 1024)
    w = eet.random_weights(cfg, 50257, seed=0)
    prompts = [[int(t) for t in np.random.default_rng(0).integers(0, 50257, size=512)]]
    _, ref = orc.generate(w, prompts, 1, 513, collect_logits=True)
    print("GPT-2-medium b1, step-0 logits vs fp32 oracle", flush=True)
    for dt, td in (("fp16", torch.float16), ("bf16", torch.bfloat16)):
        c = eet.ModelConfig(1, 1024, 24, 16, 512, 1024, datatype_label=dt)
        tr = eet.RunTrace(collect_logits=True)
        eet.generate(w, eet.GenerationRequest(prompts=prompts, steps=1), c, trace=tr)
        stats(tr.step_logits[0], ref[0], f"{dt} kernels")
        x = torch.from_numpy(w.token_embedding[prompts[0]] + w.position_embedding[:512]).cuda()[None]
        for lw in w.layers:
            x = emu_layer(x, lw, [0], 16, td)
        hl = torch.nn.functional.layer_norm(x[:, -1], (1024,), eps=1e-5).to(td) @ torch.from_numpy(w.output_head).cuda().to(td)
        stats(hl.float().cpu().numpy(), ref[0], f"{dt} torch emulation")


def c5():
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from test_baseline_layers_gpu import _fast_layer, _rows
    h, heads, s = 12288, 96, 2048
    w = _fast_layer(eet, h, 50)
    x = np.random.default_rng(51).standard_normal(size=(1, s, h), dtype=np.float32)
    rows = _rows(s, 52)
    ref = orc.decoder_layer_rows(x, w, (0,), heads, rows)
    print("c5 layer rows vs fp32 oracle", flush=True)
    for dt, td in (("fp16", torch.float16), ("bf16", torch.bfloat16)):
        cfg = eet.ModelConfig(1, h, 1, heads, s, s, datatype_label=dt)
        kv, acts = eet.preallocate_caches(cfg)
        out = eet.decoder_layer_forward(x.copy(), w, kv, eet.make_batch([s]), eet.Phase.PROMPT_PARALLEL,
                                        eet.BufferPool(), acts, 0)
        stats(out[0, rows], ref[0], f"{dt} kernels")
        for j, r in enumerate(rows):
            e = np.abs(out[0, r] - ref[0, j]).max()
            print(f"    row {r}: max abs err {e:.4f}")
        emu = emu_layer(torch.from_numpy(x).cuda(), w, [0], heads, td)[0, rows].cpu().numpy()
        stats(emu, ref[0], f"{dt} torch emulation")
        del kv, acts
        torch.cuda.empty_cache()


if __name__ == "__main__":
    which = sys.argv[1:] or ["gpt2m", "c5"]
    for n in which:
        globals()[n]()
