#!/usr/bin/env python3
"""Benchmark of the B200-native EET decoder path (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload c2|c1|c3|c4|c5] [--batch B]

Default workload (BASELINE.json configs[1], the metric's GPT-2-medium case):
GPT-2-medium shape (h=1024, 24 layers, 16 heads, vocab 50257, s_max 1024),
fp16, 16 prompts of 512 tokens + 512 greedy tokens through the public
``generate`` API. One "step" = one full generate call (prompt pass + 512
decode steps). ``value`` = generated tokens/s over the K timed steps, device
time (CUDA events, max over ranks); ``e2e`` = the same through the public API
by wall clock including the pinned H2D prompt copy and D2H token read.

Multi-GPU (torchrun, one process per GPU): each rank runs its own batch
(batch-sharded data parallelism, no collective on the data path); value =
all ranks' tokens / max-over-ranks time ("scaling": "weak").

Per-kernel roofline numbers come from a profiled replay of one step (eager,
every launch bracketed by CUDA events on its launching stream, tagged with
its algorithmic bytes/flops by the C ABI profiler). The CPU baseline times
the oracle port of the reference path (oracle/, numpy + OpenBLAS on all host
cores) on a bounded sample and extrapolates (stated in the output).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = None
try:
    with open(os.path.join(ROOT, "BASELINE.json")) as fh:
        METRIC = json.load(fh)["metric"]
except Exception:
    METRIC = "decoder-layer tokens/s at h768-12288, s<=4096; GPT-2-med 512-tok gen latency"

WORKLOADS = {
    # name: (hidden, layers, heads, vocab, prompt lengths spec, steps, dtype, batch)
    "c2": dict(hidden=1024, layers=24, heads=16, vocab=50257, prompt=512, steps=512,
               max_seq=1024, dtype="fp16", batch=16,
               desc="GPT-2 medium (h1024, 24L, 16 heads, V50257), prompt 512 + greedy 512, fp16"),
    "c1": dict(hidden=768, layers=1, heads=12, batch=4, prompt=64, dtype="fp32", kind="layer",
               lengths="ratio0.2", padding_side="right",
               desc="decoder layer h768 12 heads b4 s64, right-padded (pad ratio 0.2), fp32"),
    "c3": dict(hidden=2048, layers=1, heads=16, batch=32, prompt=1024, dtype="bf16", kind="layer",
               lengths="ragged3", desc="decoder layer h2048 16 heads s1024 b32 ragged, bf16"),
    "c4": dict(hidden=4096, layers=1, heads=32, batch=8, prompt=4096, dtype="bf16", kind="layer",
               lengths="full", desc="decoder layer h4096 32 heads s4096 b8 context phase, bf16"),
    "c5": dict(hidden=12288, layers=1, heads=96, batch=1, prompt=2048, dtype="bf16", kind="layer",
               lengths="full", tp_ok=True, desc="decoder layer h12288 96 heads s2048 b1, bf16"),
}

E2E_DEPTH = 3          # layer workloads: steps in flight in the e2e measurement (copy/compute overlap)
HBM_KINDS = {"attn_decode", "gemv", "layernorm", "embed", "argmax", "softmax", "advance", "decode_step"}


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            p = json.load(fh)
        return p["hbm_gbs"], p.get("bf16_tflops_sustained", p["bf16_tflops"]), "measured"
    except Exception:
        return 6650.0, 1400.0, "fallback (B200_PROFILING.md)"


def lengths_for(w):
    from paper_2104_12470_b200.report import prompt_lengths_for_ratio
    b, s = w["batch"], w["prompt"]
    spec = w.get("lengths", "full")
    if spec == "full":
        return [s] * b
    if spec == "ratio0.2":
        return prompt_lengths_for_ratio(b, s, 0.2)
    if spec == "ragged3":
        return [s] + [int(v) for v in np.random.default_rng(3).integers(1, s + 1, b - 1)]
    raise ValueError(spec)


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for ln in self.proc.stdout:
            self.lines.append(ln.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def mark(self):
        """index of the next sample (region bookkeeping)"""
        return len(self.lines)

    def summary(self, lo=0, hi=None):
        """samples [lo, hi) (the timed region); falls back to the samples
        adjacent to the region when it was shorter than the sampling period"""
        hi = len(self.lines) if hi is None else hi
        if hi <= lo:
            lo, hi = max(0, lo - 1), min(len(self.lines), lo + 1)
        return self._summary(self.lines[lo:hi])

    def _summary(self, lines):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for n, v in zip(names, parts[4:8]):
                if v.lower() == "active":
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        loaded = [v for v in sm if v > 0.5 * max(sm)] or sm
        return {"sm_mhz": statistics.median(loaded), "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


# --------------------------------------------------------------- CPU side
def cpu_threads():
    try:
        from threadpoolctl import threadpool_info
        return max([i.get("num_threads", 1) for i in threadpool_info()] + [1])
    except Exception:
        return os.cpu_count() or 1


def cpu_generate_sample(w, reps: int = 1):
    """Bounded sample of the reference path (oracle port, numpy + OpenBLAS on
    all cores) for the generate workload, extrapolated to the full job:
    total = L * T(prompt layer) + head + steps * (L * T(step layer at the mean
    cache length) + head). Returns (tokens/s, sample description)."""
    from oracle import eet_oracle as orc
    b, h, heads, V, p, steps, L = (w["batch"], w["hidden"], w["heads"], w["vocab"], w["prompt"],
                                   w["steps"], w["layers"])
    model = orc.seeded_weights(h, 1, heads, V, w["max_seq"], 0)
    rng = np.random.default_rng(0)
    pads = (0,) * b
    x = rng.normal(0, 1, size=(b, p, h)).astype(np.float32)
    best = None
    for _ in range(reps):
        kv = orc.OracleKV(b, heads, w["max_seq"], h // heads, 1)
        t0 = time.perf_counter()
        orc.decoder_layer(x, model.layers[0], kv, pads, 0, heads)
        t_prompt = time.perf_counter() - t0
        Lmean = p + steps // 2
        kv.filled = Lmean - 1
        x1 = x[:, :1]
        t0 = time.perf_counter()
        for _ in range(3):
            orc.decoder_layer(x1, model.layers[0], kv, pads, 0, heads)
        t_step = (time.perf_counter() - t0) / 3
        t0 = time.perf_counter()
        for _ in range(3):
            np.argmax(orc.head_logits(model, x[:, -1]), axis=1)
        t_head = (time.perf_counter() - t0) / 3
        total = L * t_prompt + t_head + steps * (L * t_step + t_head)
        best = total if best is None else min(best, total)
    sample = (f"1 prompt layer (b{b} s{p}) + 3 decode layer steps at cache length {p + steps // 2} "
              f"+ 3 LM heads, extrapolated x{L} layers x{steps} steps")
    return b * steps / best, sample


def reference_module():
    """The unmodified reference (``maskfold``) installed under baseline/_ref
    (pip --target), or None when it is absent."""
    ref = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref, "maskfold")):
        return None
    if ref not in sys.path:
        sys.path.insert(0, ref)
    try:
        import maskfold
        return maskfold
    except Exception:
        return None


def ref_generate_sample(mf, w):
    """Bounded sample of the REAL reference generate path (maskfold from
    baseline/_ref: numpy + OpenBLAS on all host cores), through its own
    decoder_layer_forward / head_logits (runtime.py:217-263, :341-344):
    one prompt layer + 2 decode layer steps at the mean cache length + 2
    heads, extrapolated to L layers x steps like cpu_generate_sample."""
    b, h, heads, V, p, steps, L = (w["batch"], w["hidden"], w["heads"], w["vocab"], w["prompt"],
                                   w["steps"], w["layers"])
    cfg = mf.ModelConfig(batch_size=b, hidden_size=h, layer_count=1, head_count=heads, max_prompt=p,
                         max_sequence=w["max_seq"])
    model = mf.random_weights(cfg, V, 0)
    kv, acts = mf.preallocate_caches(cfg)
    pool = mf.BufferPool()
    desc = mf.make_batch([p] * b)
    x = np.random.default_rng(0).normal(0, 1, size=(b, p, h)).astype(np.float32)
    t0 = time.perf_counter()
    mf.decoder_layer_forward(x, model.layers[0], kv, desc, mf.Phase.PROMPT_PARALLEL, pool, acts, 0)
    t_prompt = time.perf_counter() - t0
    Lmean = p + steps // 2
    kv.advance(Lmean - 1 - kv.filled)
    x1 = np.ascontiguousarray(x[:, :1])
    t0 = time.perf_counter()
    for _ in range(2):
        mf.decoder_layer_forward(x1.copy(), model.layers[0], kv, desc, mf.Phase.INCREMENTAL, pool, acts, 0)
    t_step = (time.perf_counter() - t0) / 2
    t0 = time.perf_counter()
    for _ in range(2):
        np.argmax(mf.runtime.head_logits(model, x[:, -1]), axis=1)
    t_head = (time.perf_counter() - t0) / 2
    total = L * t_prompt + t_head + steps * (L * t_step + t_head)
    sample = (f"reference maskfold (baseline/_ref): 1 prompt layer (b{b} s{p}) + 2 decode layer steps at "
              f"cache length {Lmean} + 2 LM heads, extrapolated x{L} layers x{steps} steps")
    return b * steps / total, sample


def ref_layer_sample(mf, w):
    """One PROMPT_PARALLEL layer of the REAL reference (maskfold), bounded
    like cpu_layer_sample (one sequence, scaled, when the batch is large)."""
    lens = lengths_for(w)
    b, h, heads = w["batch"], w["hidden"], w["heads"]
    if b * max(lens) * h > 16 * 1024 * 1024 or h >= 4096:
        lens1, scaled = [max(lens)], True
        if h >= 4096:                                  # keep the sample in the 10-30 s range
            lens1 = [min(max(lens), 1024 if h <= 4096 else 512)]
    else:
        lens1, scaled = lens, False
    s = max(lens1)
    cfg = mf.ModelConfig(batch_size=len(lens1), hidden_size=h, layer_count=1, head_count=heads, max_prompt=s,
                         max_sequence=s)
    # N(0, 0.02^2) float32 draws (the reference's float64 init takes ~1 min at
    # h12288; values do not change the time), reference field order
    rng = np.random.default_rng(0)
    mat = lambda *sh: rng.standard_normal(size=sh, dtype=np.float32) * np.float32(0.02)  # noqa: E731
    one, zero = np.ones(h, np.float32), np.zeros(h, np.float32)
    lw = mf.LayerWeights(one, zero, mat(h, h), mat(h, h), mat(h, h), mat(h, h), one.copy(), zero.copy(),
                         mat(h, 4 * h), mat(4 * h, h))
    kv, acts = mf.preallocate_caches(cfg)
    desc = mf.make_batch(lens1)
    x = np.random.default_rng(1).normal(0, 1, size=(len(lens1), s, h)).astype(np.float32)
    dt = None
    for _ in range(3 if sum(lens1) * h < 4 * 1024 * 1024 else 1):   # small samples: best of 3
        t0 = time.perf_counter()
        mf.decoder_layer_forward(x.copy(), lw, kv, desc, mf.Phase.PROMPT_PARALLEL, mf.BufferPool(), acts, 0)
        d = time.perf_counter() - t0
        dt = d if dt is None else min(dt, d)
    sample = f"reference maskfold (baseline/_ref): one layer over {len(lens1)} sequence(s) of {s}" + (
        f", scaled to the {b} x {max(lens)} workload by valid-token rate" if scaled else "")
    return sum(lens1) / dt, sample


def cpu_baseline_sample(w):
    """(tokens/s, sample, kind): the real reference when installed, else the
    oracle port of it."""
    mf = reference_module()
    kind = w.get("kind", "generate")
    if mf is not None:
        # warm numpy / OpenBLAS threads outside the sample (first call ~1 s)
        wcfg = mf.ModelConfig(batch_size=1, hidden_size=64, layer_count=1, head_count=4, max_prompt=16,
                              max_sequence=16)
        wkv, wacts = mf.preallocate_caches(wcfg)
        mf.decoder_layer_forward(np.ones((1, 16, 64), np.float32), mf.random_weights(wcfg, 8, 0).layers[0], wkv,
                                 mf.make_batch([16]), mf.Phase.PROMPT_PARALLEL, mf.BufferPool(), wacts, 0)
        v, sample = ref_generate_sample(mf, w) if kind == "generate" else ref_layer_sample(mf, w)
        return v, sample, "reference"
    v, sample = cpu_generate_sample(w) if kind == "generate" else cpu_layer_sample(w)
    return v, sample, "port"


def cpu_layer_sample(w):
    """One PROMPT_PARALLEL decoder layer on the oracle port: valid tokens/s."""
    from oracle import eet_oracle as orc
    lens = lengths_for(w)
    b, h, heads = w["batch"], w["hidden"], w["heads"]
    if b * max(lens) * h > 64 * 1024 * 1024 or h >= 4096:
        # bounded: time one sequence and scale linearly (sequences independent)
        lens1 = [max(lens)]
        scale_b = sum(lens) / max(lens)
    else:
        lens1, scale_b = lens, 1.0
    pads = orc.left_pads(lens1)
    s = max(lens1)
    model = orc.seeded_weights(h, 1, heads, 8, s, 0)
    x = np.random.default_rng(1).normal(0, 1, size=(len(lens1), s, h)).astype(np.float32)
    kv = orc.OracleKV(len(lens1), heads, s, h // heads, 1)
    t0 = time.perf_counter()
    orc.decoder_layer(x, model.layers[0], kv, pads, 0, heads)
    dt = time.perf_counter() - t0
    sample = f"one layer over {len(lens1)} sequence(s) of {s}" + (
        f", scaled linearly to {b} sequences" if scale_b != 1.0 else "")
    return sum(lens1) / dt, sample          # time is linear in tokens: same rate


def measure_fp32_peak(torch):
    torch.backends.cuda.matmul.allow_tf32 = False
    a = torch.randn(8192, 8192, device="cuda")
    b = torch.randn(8192, 8192, device="cuda")
    best = 0.0
    for _ in range(6):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        torch.matmul(a, b)
        e1.record()
        torch.cuda.synchronize()
        best = max(best, 2 * 8192 ** 3 / (e0.elapsed_time(e1) / 1e3) / 1e12)
    del a, b
    return best


def ablation_roofline(step, args, ms_full, w, hbm, torch, _lib):
    """In-graph cost of the decode kernels with programmatic dependent launch
    intact: the generate time with a kernel class left out of every decode
    step (eet_debug_skip) subtracted from the full time. Returns
    {class: (delta ms per generate, algorithmic bytes per generate, launches)}."""
    h, L, V, es, b = w["hidden"], w["layers"], w["vocab"], 2, w["batch"]
    steps, p = w["steps"], w["prompt"]
    kv = sum(b * 2 * h * es * L * (p + s + 1) for s in range(steps))
    if os.environ.get("EET_QKV_ATTN_O", "1") != "0" and h in (512, 1024) and b % 8 == 0:
        classes = {
            # decode FFN projections (gemv_cl): W1 (+LN2, GELU), W2 (+residual)
            "gemv_cl": ("w1,w2", steps * L * 8 * h * h * es, steps * L * 2),
            # LN1 + QKV + attention + out-projection in one kernel (qkv_attn_o.cu):
            # every cached K/V row of the batch + W_qkv + W_o once per step
            "qkv_attn_o": ("qkv,attn,o", kv + steps * L * 4 * h * h * es, steps * L),
            "lm_head": ("head", steps * V * h * es, steps),
        }
    elif os.environ.get("EET_ATTN_O", "1") != "0":
        classes = {
            # decode projections (gemv_cl): QKV (+LN1), W1 (+LN2, GELU), W2 (+residual)
            "gemv_cl": ("qkv,w1,w2", steps * L * 11 * h * h * es, steps * L * 3),
            # decode attention fused with the out-projection (attn_o.cu): every
            # cached K/V row of the batch + W_o once per step
            "attn_o": ("attn,o", kv + steps * L * h * h * es, steps * L),
            # LM head + fused argmax
            "lm_head": ("head", steps * V * h * es, steps),
        }
    else:
        classes = {
            "gemv_cl": ("qkv,o,w1,w2", steps * L * 12 * h * h * es, steps * L * 4),
            "attn_decode": ("attn", kv, steps * L),
            "lm_head": ("head", steps * V * h * es, steps),
        }
    out = {}
    reps = max(2, min(args.steps, 3))
    for name, (spec, byts, launches) in classes.items():
        _lib.call("eet_debug_skip", spec.encode())
        try:
            step()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(reps):
                step()
            e1.record()
            torch.cuda.synchronize()
        finally:
            _lib.call("eet_debug_skip", b"")
        delta = ms_full - e0.elapsed_time(e1) / reps
        out[name] = (delta, byts, launches)
    return out


# ------------------------------------------------------------------ main
def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def run_reference(args, w, ws, rank):
    if rank != 0:
        return
    reps = []
    sample, ckind = "", "port"
    for i in range(args.warmup + args.steps):
        v, sample, ckind = cpu_baseline_sample(w)
        if i >= args.warmup:
            reps.append(v)
    value = statistics.median(reps)
    cores = cpu_threads()
    unit = "tokens/s"
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": unit, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic (seeded random weights and tokens)",
        "config": {"workload": w["desc"], "batch_per_gpu": w["batch"],
                   "reference_compute": "float32 numpy (the reference has no 16-bit mode, core.py:20)"},
        "cpu_baseline": {"value": value, "unit": unit, "cores": cores, "kind": ckind,
                         "sample": sample},
        "e2e": {"value": value, "unit": unit, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", choices=sorted(WORKLOADS), default="c2")
    ap.add_argument("--batch", type=int, default=None)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-profile", action="store_true")
    ap.add_argument("--dp", choices=["weak", "strong"], default=None,
                    help="layer workloads under torchrun: 'strong' shards the workload's batch over the ranks "
                         "(default for c4), 'weak' gives every rank the whole batch")
    ap.add_argument("--tp", type=int, default=0,
                    help="tensor-parallel layer over the ranks (default: on for c5 under torchrun); "
                         "--tp 1 runs the sharded path on one GPU")
    args = ap.parse_args()
    w = dict(WORKLOADS[args.workload])
    if args.batch:
        w["batch"] = args.batch
    if args.dp is None:
        args.dp = "strong" if args.workload == "c4" else "weak"
    ws, rank, local = dist_env()
    args.gpus = ws if ws > 1 else args.gpus
    if args.impl == "reference":
        return run_reference(args, w, ws, rank)

    import torch
    torch.cuda.set_device(local)
    if ws > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_2104_12470_b200 as eet
    from paper_2104_12470_b200 import _lib

    kind = w.get("kind", "generate")
    hbm, tflops, peak_src = peaks()
    if w["dtype"] == "fp32":
        # fp32 mode computes at fp32 accuracy (3xTF32 on the tensor cores,
        # FFMA for decode rows; no plain TF32): its roofline
        # is the FP32 peak, not in MEASURED_PEAKS.json, so measured here:
        # cuBLAS fp32 GEMM with TF32 off (SURVEY §8(d) protocol), best of 5
        # at 8192^3
        tflops, peak_src = measure_fp32_peak(torch), "measured: torch.matmul fp32, allow_tf32=False, 8192^3"
    if kind == "generate":
        cfg = eet.ModelConfig(batch_size=w["batch"], hidden_size=w["hidden"], layer_count=w["layers"],
                              head_count=w["heads"], max_prompt=w["prompt"], max_sequence=w["max_seq"],
                              datatype_label=w["dtype"])
        weights = eet.random_weights(cfg, w["vocab"], seed=0)
        rng = np.random.default_rng(rank)
        prompts = [[int(t) for t in rng.integers(0, w["vocab"], size=w["prompt"])] for _ in range(w["batch"])]
        req = eet.GenerationRequest(prompts=prompts, steps=w["steps"])
        pool = eet.BufferPool()
        units = w["batch"] * w["steps"]            # generated tokens per step
        h2d, d2h = w["batch"] * w["prompt"] * 4, w["batch"] * w["steps"] * 8

        def step(graph=True):
            return eet.generate(weights, req, cfg, pool=pool, use_graph=graph)
    elif args.tp or (w.get("tp_ok") and ws > 1):
        # Megatron tensor parallelism: every rank holds
        # heads/tp heads and 4h/tp FFN columns; two NCCL all-reduces per
        # layer. Strong scaling: all ranks process the same tokens.
        from paper_2104_12470_b200.tp import TensorParallelLayer, shard_config
        tp = ws if ws > 1 else 1
        lens = lengths_for(w)
        desc = eet.make_batch(lens)
        s = desc.seq_len
        cfg = eet.ModelConfig(batch_size=w["batch"], hidden_size=w["hidden"], layer_count=1,
                              head_count=w["heads"], max_prompt=s, max_sequence=s,
                              datatype_label=w["dtype"])
        lw = eet.random_weights(eet.ModelConfig(1, w["hidden"], 1, w["heads"], 1, 1), 8, seed=0).layers[0]
        pool = eet.BufferPool()
        noop = (lambda t: None) if tp == 1 else None
        layer = TensorParallelLayer(lw, cfg, rank, tp, pool, all_reduce=noop)
        kv, _ = eet.preallocate_caches(shard_config(cfg, tp))
        x_host = np.random.default_rng(1).normal(0, 1, size=(w["batch"], s, w["hidden"])).astype(np.float32)
        x_dev = torch.from_numpy(x_host).cuda()
        x_pin = torch.from_numpy(x_host).pin_memory()
        out_pin = torch.empty_like(x_pin).pin_memory()
        units = sum(lens)
        h2d = d2h = x_host.nbytes
        w["desc"] = w["desc"] + f", tensor-parallel tp{tp}"
        w["tp"] = tp

        def step(graph=True, host=False):
            kv._filled = 0
            if host:
                xd = x_pin.to("cuda", non_blocking=True)
                layer.forward(xd, kv, desc, _lib.PHASE_PROMPT, 0)
                return out_pin.copy_(xd, non_blocking=True)
            return layer.forward(x_dev, kv, desc, _lib.PHASE_PROMPT, 0)
    else:
        lens = lengths_for(w)
        if ws > 1 and args.dp == "strong":
            # batch-sharded data parallelism: the workload's
            # sequences split over the ranks by causal cost, no collective
            from paper_2104_12470_b200.dp import shard_lengths
            mine = shard_lengths(lens, ws)[rank]
            lens = [lens[i] for i in mine] or [1]
            w["batch"] = len(lens)
            w["dp_strong"] = True
        # BASELINE configs[0] (c1) is right-padded: native valid windows [0, len_b)
        side = w.get("padding_side", "left")
        desc = eet.make_batch(lens, padding_side=side)
        s = desc.seq_len
        cfg = eet.ModelConfig(batch_size=w["batch"], hidden_size=w["hidden"], layer_count=1,
                              head_count=w["heads"], max_prompt=s, max_sequence=s,
                              datatype_label=w["dtype"])
        lw = eet.random_weights(eet.ModelConfig(1, w["hidden"], 1, w["heads"], 1, 1), 8, seed=0).layers[0]
        kv, acts = eet.preallocate_caches(cfg)
        pool = eet.BufferPool()
        x_host = np.random.default_rng(1).normal(0, 1, size=(w["batch"], s, w["hidden"])).astype(np.float32)
        x_dev = torch.from_numpy(x_host).cuda()
        x_pin = torch.from_numpy(x_host).pin_memory()
        out_pin = torch.empty_like(x_pin).pin_memory()
        units = sum(lens)
        # heavily padded batches (c3: 44% valid) copy only each sequence's
        # valid slots [start, end); otherwise one copy of the whole array
        windows = desc.windows() if units * w["hidden"] * 4 < 0.7 * x_host.nbytes else None
        h2d = d2h = units * w["hidden"] * 4 if windows else x_host.nbytes

        # e2e: every step copies its valid hidden-state rows pinned host -> device, runs
        # the layer through the public API and copies the result back to
        # pinned host memory. E2E_DEPTH independent contexts (stream, K/V
        # cache, buffer pool, device buffer) take the steps in turn, so one
        # step's host->device copy, another's layer and a third's
        # device->host copy overlap (the two copy engines and the SMs are
        # separate resources) -- how a server keeps the GPU busy between
        # requests.
        ctxs = []
        for i in range(E2E_DEPTH):
            kv_i, acts_i = (kv, acts) if i == 0 else eet.preallocate_caches(cfg)
            ctxs.append({"s": torch.cuda.Stream(), "kv": kv_i, "acts": acts_i,
                         "pool": pool if i == 0 else eet.BufferPool(), "x": torch.empty_like(x_dev),
                         "out": torch.empty_like(x_pin).pin_memory()})
        host_i = [0]

        def step(graph=True, host=False):
            if host:
                c = ctxs[host_i[0] % len(ctxs)]
                host_i[0] += 1
                with torch.cuda.stream(c["s"]):
                    c["kv"]._filled = 0
                    if windows is None:
                        c["x"].copy_(x_pin, non_blocking=True)
                    else:                                          # valid rows only: pad rows are
                        for i, (a0, a1) in enumerate(windows):     # never read ...
                            c["x"][i, a0:a1].copy_(x_pin[i, a0:a1], non_blocking=True)
                    eet.decoder_layer_forward(c["x"], lw, c["kv"], desc, eet.Phase.PROMPT_PARALLEL, c["pool"],
                                              c["acts"], 0)
                    if windows is None:
                        c["out"].copy_(c["x"], non_blocking=True)
                    else:                                          # ... nor written by the layer
                        for i, (a0, a1) in enumerate(windows):
                            c["out"][i, a0:a1].copy_(c["x"][i, a0:a1], non_blocking=True)
                return c["out"]
            kv._filled = 0
            return eet.decoder_layer_forward(x_dev, lw, kv, desc, eet.Phase.PROMPT_PARALLEL, pool, acts, 0)

    clk = ClockSampler(torch.cuda.current_device()).__enter__()   # running before the warm-up
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if ws > 1:
        dist.barrier()
    launches0 = _lib.launch_count()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    clk_lo = clk.mark()
    ev0.record()
    for _ in range(args.steps):
        step()
    ev1.record()
    torch.cuda.synchronize()
    clk_hi = clk.mark()
    clk.__exit__(None, None, None)
    launches = _lib.launch_count() - launches0
    ms = ev0.elapsed_time(ev1)
    if ws > 1:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        dist.barrier()
    tp_mode = bool(w.get("tp"))
    strong = tp_mode or bool(w.get("dp_strong"))
    if w.get("dp_strong"):                    # ranks hold different shards: sum of valid tokens
        tot = torch.tensor([float(units)], device="cuda")
        dist.all_reduce(tot)
        units_all = tot.item()
    else:
        units_all = units * (1 if tp_mode else ws)
    value = units_all * args.steps / (ms / 1e3)

    # end to end through the public API: host inputs in, host results out
    if kind != "generate" and not tp_mode:
        for _ in range(E2E_DEPTH):                 # first use of every context outside the timing
            step(host=True)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step(host=True) if kind != "generate" else step()
    torch.cuda.synchronize()
    e2e_s = time.perf_counter() - t0
    if ws > 1:
        t = torch.tensor([e2e_s], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    e2e = units_all * args.steps / e2e_s

    extra = {}
    if kind == "generate" and rank == 0:
        # batch-1 latency of the same workload (BASELINE c2 also quotes b=1)
        cfg1 = eet.ModelConfig(1, w["hidden"], w["layers"], w["heads"], w["prompt"], w["max_seq"],
                               datatype_label=w["dtype"])
        req1 = eet.GenerationRequest(prompts=prompts[:1], steps=w["steps"])
        eet.generate(weights, req1, cfg1, pool=pool)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        eet.generate(weights, req1, cfg1, pool=pool)
        torch.cuda.synchronize()
        extra["latency_b1_s"] = time.perf_counter() - t0

    roofline, kernels, ablation = None, {}, {}
    if not args.no_profile and rank == 0:
        # per-kernel view from a profiled replay: CUDA events around every
        # launch (in the decode graph they sit between PDL-linked kernels and
        # break the overlap, so these are per-launch upper bounds)
        _lib.profile_enable(True)
        step(graph=True)
        torch.cuda.synchronize()
        summ = _lib.profile_summary()
        _lib.profile_enable(False)
        total = sum(v[1] for v in summ.values()) or 1.0
        for name, (n, kms, by, fl) in summ.items():
            hbm_k = name in HBM_KINDS
            ach = (by / (kms / 1e3) / 1e9) if hbm_k else (fl / (kms / 1e3) / 1e12)
            kernels[name] = {"launches": n, "ms": round(kms, 4), "share": round(kms / total, 4),
                             "achieved": round(ach, 2), "unit": "GB/s" if hbm_k else "TFLOP/s",
                             "frac": round(ach / (hbm if hbm_k else tflops), 4)}
        tf = os.path.join(ROOT, "profiles", "traffic_per_launch.json")
        traffic_tab = json.load(open(tf)).get(args.workload, {}) if os.path.exists(tf) else {}
        if kind == "generate":
            # headline roofline from in-graph ablation deltas (PDL intact)
            ms_gen = ms / args.steps
            abl = ablation_roofline(step, args, ms_gen, w, hbm, torch, _lib)
            for name, (dms, byts, nl) in abl.items():
                ach = byts / (dms / 1e3) / 1e9 if dms > 0 else None
                ablation[name] = {"ms_per_generate": round(dms, 3), "share": round(dms / ms_gen, 4),
                                  "launches": nl, "avg_launch_us": round(dms / nl * 1e3, 3),
                                  "algorithmic_bytes": byts, "achieved": round(ach, 1) if ach else None,
                                  "unit": "GB/s", "frac": round(ach / hbm, 4) if ach else None}
            dom = max(ablation, key=lambda k: ablation[k]["ms_per_generate"])
            a = ablation[dom]
            roofline = {"kernel": dom, "bound": "hbm", "achieved": a["achieved"], "peak": hbm, "unit": "GB/s",
                        "frac": a["frac"], "traffic": traffic_tab.get(dom),
                        "algorithmic_per_launch": a["algorithmic_bytes"] / a["launches"],
                        "avg_launch_us": a["avg_launch_us"], "peak_source": peak_src,
                        "timing": "in-graph ablation: device time of the whole generate minus the same with "
                                  "this kernel class left out of every decode step (eet_debug_skip), CUDA events, "
                                  "PDL intact; avg_launch_us = that delta / launches"}
        else:
            dom = max(summ, key=lambda k: summ[k][1])
            n, kms, by, fl = summ[dom]
            hbm_k = dom in HBM_KINDS
            ach = kernels[dom]["achieved"]
            roofline = {"kernel": dom, "bound": "hbm" if hbm_k else "tensor", "achieved": ach,
                        "peak": hbm if hbm_k else tflops, "unit": "GB/s" if hbm_k else "TFLOP/s",
                        "frac": round(ach / (hbm if hbm_k else tflops), 4), "traffic": traffic_tab.get(dom),
                        "algorithmic_per_launch": (by if hbm_k else fl) / n,
                        "avg_launch_us": kms / n * 1e3, "peak_source": peak_src,
                        "timing": "profiled replay of one layer: CUDA events around every launch on its stream"}

    # whole-generate HBM roofline (c2): every decode step must stream all
    # weights once (+ LM head) and every cached K/V row of the batch once
    step_roofline = None
    if kind == "generate":
        h_, L_, V_, es_ = w["hidden"], w["layers"], w["vocab"], 2
        wbytes = (12 * h_ * h_ * L_ + V_ * h_) * es_
        kv = sum(w["batch"] * 2 * h_ * es_ * L_ * (w["prompt"] + s + 1) for s in range(w["steps"]))
        byts = w["steps"] * wbytes + kv
        ach = byts / (ms / args.steps / 1e3) / 1e9
        step_roofline = {"bound": "hbm", "algorithmic_bytes_per_generate": byts, "achieved": round(ach, 1),
                         "peak": hbm, "unit": "GB/s", "frac": round(ach / hbm, 4),
                         "note": "decode steps' weight + KV bytes over the device time of the whole generate "
                                 "(prompt pass included in the time)"}

    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        v, sample, ckind = cpu_baseline_sample(w)
        cpu = {"value": v, "unit": "tokens/s", "cores": cpu_threads(), "kind": ckind, "sample": sample}

    if rank == 0:
        clocks = clk.summary(clk_lo, clk_hi)
        line = {
            "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
            "scaling": "strong" if strong else "weak", "vs_baseline": None,
            "dtype": {"fp16": "f16", "bf16": "bf16", "fp32": "f32"}[w["dtype"]],
            "data": "synthetic (seeded random weights N(0,0.02), random token ids / hidden states)",
            "config": {"workload": w["desc"], "batch_per_gpu": w["batch"],
                       "parallelism": f"tp{w['tp']}" if tp_mode else (
                           (f"dp{ws} batch-sharded" if w.get("dp_strong") else f"dp{ws} replicated batch")
                           if ws > 1 else "single"),
                       "l2": "working set (weights+KV) > 126 MB L2 every step; no flush needed",
                       "tokens_per_step": units},
            "e2e": {"value": e2e, "unit": "tokens/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
            "gpu_launches": int(launches),
            "clocks": clocks,
            "roofline": roofline,
            "cpu_baseline": cpu,
            "kernels": kernels,
        }
        if ablation:
            line["kernels_in_graph"] = ablation
        if step_roofline:
            line["generate_roofline"] = step_roofline
        line.update(extra)
        print(json.dumps(line), flush=True)
    if ws > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
