"""Fused decode kernels through the layer API: prompt pass + incremental
steps against the fp32 oracle, and bit-identical repeats (the heads'
out-projection contributions are summed as 2^-32 fixed-point integer
atomics, so their arrival order cannot change the result).

* GPT-2-medium width at b16 (fp16, bf16): LayerNorm 1 + QKV + attention +
  out-projection in one kernel (csrc/qkv_attn_o.cu; hidden 512/1024,
  clusters of 8 sequences, split-K QKV over the cluster);
* h2048 / 32 heads at b8 (bf16): attention + out-projection (csrc/attn_o.cu,
  256 W_o rows per CTA, two row tiles per warp) after the QKV GEMV.

Reference: /root/reference/pkg/src/maskfold/runtime.py:160-188 (attention,
context @ W_o into the residual), :217-263 (the layer).
"""

import numpy as np
import pytest

from conftest import check_16bit

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def eet(cuda_ok):
    import paper_2104_12470_b200 as m
    return m


def _layer(eet, h, seed):
    rng = np.random.default_rng(seed)

    def draw(*shape):
        a = rng.standard_normal(size=shape, dtype=np.float32)
        a *= np.float32(0.02)
        return a

    g = (1.0 + 0.1 * rng.standard_normal(h)).astype(np.float32)
    b = (0.1 * rng.standard_normal(h)).astype(np.float32)
    return eet.LayerWeights(g, b, draw(h, h), draw(h, h), draw(h, h), draw(h, h),
                            g.copy(), b.copy(), draw(h, 4 * h), draw(4 * h, h))


def _run(eet, w, cfg, desc, x, steps_x):
    kv, acts = eet.preallocate_caches(cfg)
    pool = eet.BufferPool()
    s = desc.seq_len
    eet.decoder_layer_forward(x.copy(), w, kv, desc, eet.Phase.PROMPT_PARALLEL, pool, acts, 0)
    kv.advance(s)
    outs = []
    for sx in steps_x:
        outs.append(np.asarray(eet.decoder_layer_forward(sx.copy(), w, kv, desc, eet.Phase.INCREMENTAL, pool,
                                                         acts, 0)))
        kv.advance(1)
    return outs


@pytest.mark.parametrize("h,heads,b,bmax,dt", [(1024, 16, 16, 16, "fp16"), (1024, 16, 16, 16, "bf16"),
                                               (1024, 16, 8, 16, "fp16"), (2048, 32, 8, 8, "bf16")])
def test_fused_decode_steps_vs_oracle(eet, h, heads, b, bmax, dt):
    """bmax: the configuration's batch (capacity); b < bmax runs one cluster
    of 8 sequences per head on a runtime sized for 16."""
    from oracle import eet_oracle as orc
    s, nsteps = 96, 3
    rng = np.random.default_rng(h + b)
    lengths = [s] + [int(n) for n in rng.integers(1, s + 1, size=b - 1)]
    desc = eet.make_batch(lengths)
    w = _layer(eet, h, 7)
    cfg = eet.ModelConfig(batch_size=bmax, hidden_size=h, layer_count=1, head_count=heads, max_prompt=s,
                          max_sequence=s + nsteps, datatype_label=dt)
    x = rng.standard_normal(size=(b, s, h), dtype=np.float32)
    steps_x = [rng.standard_normal(size=(b, 1, h), dtype=np.float32) for _ in range(nsteps)]
    outs = _run(eet, w, cfg, desc, x, steps_x)

    pads = tuple(desc.padding_len)
    okv = orc.OracleKV(b, heads, s + nsteps, h // heads, 1)
    orc.decoder_layer(x, w, okv, pads, 0, heads)
    okv.advance(s)
    for i, sx in enumerate(steps_x):
        ref = orc.decoder_layer(sx, w, okv, pads, 0, heads)
        okv.advance(1)
        check_16bit(outs[i], ref, dt, f"fused decode step {i} h{h} b{b} {dt}")

    again = _run(eet, w, cfg, desc, x, steps_x)
    for i in range(nsteps):
        assert np.array_equal(outs[i], again[i]), f"step {i} not bit-identical between runs"
