"""Run-to-run determinism of the decode path (GPT-2-medium shape, fp16):
the same greedy request repeated in one process — interleaved with other
batch sizes and bf16 runs that recycle the allocator's memory — must give
bit-identical logits and tokens every time. Catches races in the decode
kernels: the LM head's shared weight ring once let a consumer warp read a
stage two phases early (a wrong 16-row vocab tile in one step, ~1 run in 3);
the fused decode kernels sum the heads' out-projection contributions with
integer atomics precisely so that arrival order cannot matter.

Reference: runtime.py:372-437 (the reference is deterministic numpy)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def eet(cuda_ok):
    import paper_2104_12470_b200 as m
    return m


def test_generate_repeats_bit_identical(eet):
    steps = 32
    w = eet.random_weights(eet.ModelConfig(16, 1024, 24, 16, 512, 512 + steps), 50257, seed=0)

    def run(b, dt):
        cfg = eet.ModelConfig(b, 1024, 24, 16, 512, 512 + steps, datatype_label=dt)
        rng = np.random.default_rng(b)
        prompts = [[int(t) for t in rng.integers(0, 50257, size=int(n))] for n in rng.integers(400, 513, size=b)]
        tr = eet.RunTrace(collect_logits=True)
        toks = eet.generate(w, eet.GenerationRequest(prompts=prompts, steps=steps), cfg, trace=tr)
        return toks, np.stack(tr.step_logits)

    ref = {b: run(b, "fp16") for b in (1, 16)}
    for rep in range(3):
        run(16, "bf16")
        for b in (1, 16):
            toks, logits = run(b, "fp16")
            d = np.abs(logits - ref[b][1]).max(axis=(1, 2))
            assert not d.any(), f"rep {rep} b{b}: logits differ from step {int(np.argmax(d > 0))} (max {d.max():.3g})"
            assert np.array_equal(toks, ref[b][0])
