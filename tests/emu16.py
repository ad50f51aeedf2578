"""16-bit rounding budget (test infrastructure, GPU only).

A plain PyTorch restatement of the reference layer (runtime.py:106-263,
Appendix A of SURVEY.md) that rounds at exactly the points this package's
16-bit path rounds — weights, LayerNorm outputs, q/k/v, P, context and the
FFN intermediate in the 16-bit type; fp32 accumulation and an fp32
residual stream — computed by cuBLAS / torch. Its error against the fp32
oracle is what the FORMAT costs; a kernel whose error is no larger is as
accurate as the format allows. (bf16 carries 8 significant bits, fp16 11:
at GPT-2-medium depth or K = 4h = 49152 the bf16 format alone exceeds the
north-star's elementwise 2e-2 on a few elements — measured.)
"""

import math

import numpy as np
import torch


def _dev(a, td):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda().to(td)


def emu_layer(x, w, pads, heads, td):
    """x [b, t, h] fp32 cuda, prompt phase, causal attention over [pad_b, i]."""
    b, t, h = x.shape
    hd = h // heads

    def ln(v, g, bb):
        return torch.nn.functional.layer_norm(v, (h,), _dev(g, torch.float32), _dev(bb, torch.float32), 1e-5)

    l1 = ln(x, w.ln1_scale, w.ln1_shift).to(td)
    q, k, v = l1 @ _dev(w.wq, td), l1 @ _dev(w.wk, td), l1 @ _dev(w.wv, td)
    sp = lambda a: a.view(b, t, heads, hd).transpose(1, 2)  # noqa: E731
    s = (sp(q).float() @ sp(k).float().transpose(2, 3)) * (1.0 / math.sqrt(hd))
    i = torch.arange(t, device="cuda")
    pad = torch.tensor(list(pads), device="cuda")
    mask = (i[None, :] <= i[:, None])[None, None] & (i[None, None, None, :] >= pad[:, None, None, None])
    s = s.masked_fill(~mask, float("-inf"))
    p = torch.softmax(s, -1).nan_to_num(0.0).to(td)
    del s
    ctx = (p @ sp(v)).transpose(1, 2).reshape(b, t, h).to(td)
    x = x + (ctx @ _dev(w.wo, td)).float()
    l2 = ln(x, w.ln2_scale, w.ln2_shift).to(td)
    mid = (l2 @ _dev(w.w1, td)).float()
    mid = (mid * 0.5 * (1 + torch.tanh(math.sqrt(2 / math.pi) * (mid + 0.044715 * mid ** 3)))).to(td)
    return x + (mid @ _dev(w.w2, td)).float()


def emu_layer_rows(x, w, pads, heads, td, rows):
    """emu_layer's output at the selected query rows, as numpy [b, len(rows), h]."""
    out = emu_layer(torch.from_numpy(np.ascontiguousarray(x)).cuda(), w, pads, heads, td)
    return out[:, list(rows)].cpu().numpy()


def emu_first_logits(model, prompts, td):
    """Step-0 logits of ``generate`` (prompt pass + final LN + LM head) for
    equal-length prompts, numpy [b, vocab]."""
    t = len(prompts[0])
    assert all(len(p) == t for p in prompts)
    tok = np.asarray(prompts)
    x = torch.from_numpy(model.token_embedding[tok] + model.position_embedding[:t][None]).cuda().float()
    heads = model.head_count
    for lw in model.layers:
        x = emu_layer(x, lw, [0] * len(prompts), heads, td)
    h = x.shape[-1]
    last = torch.nn.functional.layer_norm(x[:, -1], (h,), _dev(model.final_scale, torch.float32),
                                          _dev(model.final_shift, torch.float32), 1e-5).to(td)
    return (last @ _dev(model.output_head, td)).float().cpu().numpy()


def bound_ratio(ours, ref, rtol=2e-2):
    """max over elements of |d| / (rtol|ref| + rtol rms(ref)) — the combined
    north-star form; <= 1 passes."""
    ours, ref = np.asarray(ours, np.float64), np.asarray(ref, np.float64)
    rms = float(np.sqrt(np.mean(ref * ref)))
    return float((np.abs(ours - ref) / (rtol * np.abs(ref) + rtol * rms)).max())


def norm_rel(ours, ref):
    ours, ref = np.asarray(ours, np.float64), np.asarray(ref, np.float64)
    return float(np.linalg.norm(ours - ref) / np.linalg.norm(ref))
