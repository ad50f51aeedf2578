"""GPU parity of the operator-level kernels against the golden vectors from
the reference and the CPU oracle (test infrastructure)."""

import numpy as np
import pytest
from numpy.testing import assert_allclose

from conftest import load_golden

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def eet(cuda_ok):
    import paper_2104_12470_b200 as m
    return m


@pytest.fixture(scope="module")
def sm():
    return load_golden("softmax")


def test_causal_and_padding_softmax_golden(eet, sm):
    """attention.py:73-135 vs the reference outputs: atol 1e-6, exact zeros
    outside the window, valid rows sum to one (test_acceptance.py:56-87)."""
    for i in range(int(sm["n_cases"])):
        raw, pads, heads = sm[f"c{i}_raw"], tuple(int(p) for p in sm[f"c{i}_pads"]), int(sm[f"c{i}_heads"])
        desc = eet.BatchDescriptor(seq_len=raw.shape[1], padding_len=pads, batch=len(pads))
        for causal, op, key in ((True, eet.fused_causal_softmax, "causal"),
                                (False, eet.fused_padding_softmax, "padding")):
            out = op(eet.AttentionScores(raw.copy(), desc.batch, heads), desc).data
            ref = sm[f"c{i}_{key}"]
            assert_allclose(out, ref, atol=1e-6)
            assert np.array_equal(out == 0, ref == 0), f"case {i} {key}: zero pattern"
            for b, pad in enumerate(pads):
                planes = out[b * heads:(b + 1) * heads]
                assert np.all(np.abs(planes[:, pad:, :].sum(-1) - 1.0) <= 1e-6)


def test_step_softmax_golden(eet, sm):
    for i in range(int(sm["n_step"])):
        raw, pads = sm[f"s{i}_raw"], tuple(int(p) for p in sm[f"s{i}_pads"])
        desc = eet.BatchDescriptor(seq_len=raw.shape[2], padding_len=pads, batch=len(pads))
        out = eet.fused_step_softmax(raw.copy(), desc)
        assert_allclose(out, sm[f"s{i}_out"], atol=1e-6)
        for b, pad in enumerate(pads):
            assert np.all(out[b, :, :pad] == 0)


def test_folded_plane_1030(eet, sm):
    """seq 1030 folds into (2, 515) sub-blocks (folding.py:30-54)."""
    raw = np.random.default_rng(int(sm["big_seed"])).normal(0.0, 3.0, size=(1, 1030, 1030)).astype(np.float32)
    desc = eet.BatchDescriptor(seq_len=1030, padding_len=tuple(int(p) for p in sm["big_pads"]), batch=1)
    out = eet.fused_causal_softmax(eet.AttentionScores(raw, 1, 1), desc).data
    assert_allclose(out[0, sm["big_rows"]], sm["big_causal_rows"], atol=1e-6)


def test_tiny_fold_cap_and_large_planes(eet):
    """Forced multi-sub-block reductions (cap 3, test_attention.py:79-89) and
    a seq-4096 plane (fold (4, 1024)) against the oracle."""
    from oracle import eet_oracle as orc
    rng = np.random.default_rng(5)
    for _ in range(20):
        s = int(rng.integers(1, 17))
        pads = tuple(int(rng.integers(0, s)) for _ in range(2))
        desc = eet.BatchDescriptor(seq_len=s, padding_len=pads, batch=2)
        raw = rng.normal(0, 3, size=(4, s, s)).astype(np.float32)
        out = eet.fused_causal_softmax(eet.AttentionScores(raw.copy(), 2, 2), desc,
                                       plan=eet.plan_folding(s, unit_cap=3)).data
        assert_allclose(out, orc.masked_softmax(raw, pads, 2, True), atol=1e-6)
    s = 4096
    x = torch.randn(2, s, s, device="cuda") * 3
    desc = eet.BatchDescriptor(seq_len=s, padding_len=(0, 1000), batch=2)
    eet.fused_causal_softmax(eet.AttentionScores(x, 2, 1), desc)
    rows = [0, 999, 1000, 1001, 2047, 4095]
    host = x[:, rows].cpu().numpy()
    assert np.all(host[1, :2] == 0)                     # pad-query rows of sequence 1
    sums = x.sum(-1).cpu().numpy()
    assert np.abs(sums[0] - 1).max() < 1e-5 and np.abs(sums[1, 1000:] - 1).max() < 1e-5


def test_softmax_known_answers(eet):
    desc = eet.make_batch([3])
    s = eet.AttentionScores(np.zeros((1, 3, 3), np.float32), 1, 1)
    eet.fused_causal_softmax(s, desc)
    assert_allclose(s.data[0], [[1, 0, 0], [.5, .5, 0], [1 / 3, 1 / 3, 1 / 3]], atol=1e-6)
    desc = eet.BatchDescriptor(seq_len=4, padding_len=(2,), batch=1)
    raw = np.random.default_rng(0).normal(size=(1, 4, 4)).astype(np.float32)
    out = eet.fused_causal_softmax(eet.AttentionScores(raw, 1, 1), desc).data
    assert np.array_equal(out[0, :2], np.zeros((2, 4)))
    assert_allclose(out[0, 2], [0, 0, 1, 0], atol=1e-6)
    with pytest.raises(ValueError):
        eet.fused_causal_softmax(eet.AttentionScores(np.zeros((1, 3, 3), np.float32), 1, 1),
                                 eet.make_batch([3, 3]))
    with pytest.raises(ValueError):
        eet.fused_causal_softmax(eet.AttentionScores(np.zeros((1, 4, 4), np.float32), 1, 1),
                                 eet.make_batch([4]), plan=eet.plan_folding(8))


def test_mha_golden(eet):
    g = load_golden("mha")
    for i in range(int(g["n_cases"])):
        pads = tuple(int(p) for p in g[f"m{i}_pads"])
        q = g[f"m{i}_q"]
        desc = eet.BatchDescriptor(seq_len=q.shape[1], padding_len=pads, batch=len(pads))
        out = eet.mha_forward(q, g[f"m{i}_k"], g[f"m{i}_v"], desc, int(g[f"m{i}_heads"]),
                              causal=bool(g[f"m{i}_causal"]))
        assert_allclose(out, g[f"m{i}_out"], atol=1e-5)
        for b, pad in enumerate(pads):
            assert np.all(out[b, :pad] == 0)


def test_mha_pad_perturbation_bit_identical(eet):
    desc = eet.BatchDescriptor(seq_len=6, padding_len=(3, 1), batch=2)
    rng = np.random.default_rng(11)
    q, k, v = (rng.normal(size=(2, 6, 8)).astype(np.float32) for _ in range(3))
    for causal in (True, False):
        base = eet.mha_forward(q, k, v, desc, 2, causal=causal)
        k2, v2 = k.copy(), v.copy()
        for b, pad in enumerate(desc.padding_len):
            k2[b, :pad] = rng.normal(size=(pad, 8))
            v2[b, :pad] = rng.normal(size=(pad, 8))
        pert = eet.mha_forward(q, k2, v2, desc, 2, causal=causal)
        for b, pad in enumerate(desc.padding_len):
            assert np.array_equal(base[b, pad:], pert[b, pad:])
    one = eet.make_batch([1])
    qq, kk, vv = (np.random.default_rng(i).normal(size=(1, 1, 4)).astype(np.float32) for i in range(3))
    assert_allclose(eet.mha_forward(qq, kk, vv, one, 2), vv, atol=1e-7)


def test_layer_norm_vs_oracle(eet):
    from oracle import eet_oracle as orc
    rng = np.random.default_rng(1)
    for h in (8, 30, 768, 1024, 4096, 12288, 16384):
        x = rng.normal(0, 2, size=(5, h)).astype(np.float32)
        g = rng.normal(1, 0.1, size=h).astype(np.float32)
        b = rng.normal(0, 0.1, size=h).astype(np.float32)
        out = eet.layer_norm(x, g, b)
        assert_allclose(out, orc.layer_norm(x, g, b), atol=2e-5, rtol=1e-5)


def _gemm(dtype_code, a, b, bias=None):
    from paper_2104_12470_b200 import _lib
    td = {0: torch.float32, 1: torch.bfloat16, 2: torch.float16}[dtype_code]
    A = torch.as_tensor(a).to("cuda", td).contiguous()
    B = torch.as_tensor(b).to("cuda", td).contiguous()
    M, K = A.shape
    N = B.shape[0]
    C = torch.full((M, N), float("nan"), device="cuda")
    bias_t = torch.as_tensor(bias).cuda() if bias is not None else None
    _lib.call("eet_gemm", dtype_code, A.data_ptr(), B.data_ptr(),
              bias_t.data_ptr() if bias_t is not None else None, C.data_ptr(), M, N, K, N,
              torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    return C.cpu().numpy(), A.float().cpu().numpy(), B.float().cpu().numpy()


@pytest.mark.parametrize("M,N,K", [(1, 64, 64), (7, 100, 40), (16, 3072, 1024), (17, 50, 24),
                                   (205, 2304, 768), (300, 130, 100), (205, 768, 3072), (64, 64, 4100)])
def test_fp32_gemm_exact_path(eet, M, N, K):
    """True-fp32 GEMM (split-K with an ordered second-stage reduction for
    small M x N) against fp64."""
    rng = np.random.default_rng(M * 7 + N)
    a = rng.normal(size=(M, K)).astype(np.float32)
    b = rng.normal(size=(N, K)).astype(np.float32)
    c, _, _ = _gemm(0, a, b)
    ref = a.astype(np.float64) @ b.astype(np.float64).T
    assert np.abs(c - ref).max() <= 1e-5 * np.sqrt(K) * np.abs(ref).max() + 1e-5


@pytest.mark.parametrize("dt", [1, 2])
@pytest.mark.parametrize("M,N,K", [(128, 256, 64), (200, 384, 192), (1000, 768, 200),
                                   (4096, 3 * 2048, 2048), (257, 128, 4096), (130, 50257, 1024),
                                   (33, 1000, 8), (5, 3072, 1024), (16, 4096, 1024),
                                   (1, 50257, 1024), (24, 1024, 4096), (32, 3072, 1024),
                                   (3, 1000, 200), (2, 130, 64)])
def test_tensor_core_gemm(eet, dt, M, N, K):
    """tcgen05 GEMM (M > 32) / tcgen05 swap-AB split-K GEMV (M <= 32) vs fp64
    on the same 16-bit-rounded operands: only accumulation-order error."""
    rng = np.random.default_rng(M + N + K)
    a = rng.normal(size=(M, K)).astype(np.float32)
    b = rng.normal(size=(N, K)).astype(np.float32)
    bias = rng.normal(size=N).astype(np.float32)
    c, a16, b16 = _gemm(dt, a, b, bias)
    ref = a16.astype(np.float64) @ b16.astype(np.float64).T + bias
    err = np.abs(c - ref).max()
    assert np.isfinite(c).all(), "unwritten outputs"
    assert err <= 2e-5 * np.sqrt(K) * 4 + 1e-4, f"max err {err}"
