"""The incremental-phase projection kernel (csrc/gemv_cl.cu) through its C-ABI
test entry ``eet_gemv_decode`` against a plain PyTorch fp32 restatement of
the same op on the same 16-bit operands:

* plain:  out = X W^T                     (out-proj / W2 shape, runtime.py:188, :212)
* LN:     out = LN(x) W^T, LN in fp32 then rounded to the 16-bit type
          (QKV / W1 shape, runtime.py:83-94, :131-136, :204-209)
* GELU:   out = gelu_tanh(LN(x) W^T) stored 16-bit (runtime.py:97-103)
* resid:  out += X W^T (fp32 residual stream, runtime.py:188 / :259)

Shapes cover the cluster split (C = 8 / 6 / 4 K-slices), partial row tiles
(N % 16 != 0 is rejected by the TMA row box only through OOB zero fill),
one and two token n-blocks (M <= 8 / M <= 16) and the GPT-2-medium decode
shapes. Tolerance: fp32 accumulation-order differences only (the operands
are identical), 1e-3 of the output rms.
"""

import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

DT = {"bf16": (1, torch.bfloat16), "fp16": (2, torch.float16)}     # eet_dtype codes
MODES = {"f32": 0, "gelu": 2, "resid": 3}


@pytest.fixture(scope="module")
def lib(cuda_ok):
    from paper_2104_12470_b200 import _lib
    return _lib


def _gelu(u):
    return u * 0.5 * (1 + torch.tanh(math.sqrt(2 / math.pi) * (u + 0.044715 * u ** 3)))


def _run(lib, dt, M, N, K, mode, ln, seed):
    code, td = DT[dt]
    g = torch.Generator(device="cuda").manual_seed(seed)
    W = (torch.randn(N, K, device="cuda", generator=g) * 0.02).to(td)
    x = torch.randn(M, K, device="cuda", generator=g) * 1.5 + 0.3
    gam = torch.rand(K, device="cuda", generator=g) + 0.5
    bet = torch.randn(K, device="cuda", generator=g) * 0.1
    X = torch.randn(M, K, device="cuda", generator=g).to(td)
    if ln:
        inp = torch.nn.functional.layer_norm(x, (K,), gam, bet, 1e-5).to(td)
    else:
        inp = X
    ref = inp.float() @ W.float().t()
    st = torch.cuda.current_stream().cuda_stream
    if mode == "gelu":
        out = torch.empty(M, N, device="cuda", dtype=td)
        ref = _gelu(ref).to(td).float()
    elif mode == "resid":
        base = torch.randn(M, N, device="cuda", generator=g)
        out = base.clone()
        ref = ref + base
    else:
        out = torch.empty(M, N, device="cuda", dtype=torch.float32)
    lib.call("eet_gemv_decode", code, W.data_ptr(), N, K, 0 if ln else X.data_ptr(),
             x.data_ptr() if ln else 0, gam.data_ptr() if ln else 0, bet.data_ptr() if ln else 0,
             M, MODES[mode], out.data_ptr(), st)
    torch.cuda.synchronize()
    return out.float(), ref


SHAPES = [
    # M, N, K
    (16, 3072, 1024),     # GPT-2-medium QKV, b16
    (16, 1024, 1024),     # out-proj
    (16, 4096, 1024),     # W1
    (16, 1024, 4096),     # W2 (Kc = 512)
    (1, 1024, 1024),      # b1
    (9, 2304, 768),       # C = 6 slices, two n-blocks
    (3, 200, 256),        # C = 4, partial last cluster
    (8, 8192, 2048),      # Kc = 256, more clusters than SMs / 8
    (5, 48, 512),         # one cluster
    (2, 96, 64),          # K = 64: a one-CTA cluster (C = 1)
]


@pytest.mark.parametrize("dt", ["fp16", "bf16"])
@pytest.mark.parametrize("M,N,K", SHAPES)
def test_plain_projection(lib, dt, M, N, K):
    out, ref = _run(lib, dt, M, N, K, "f32", False, M * 7 + N)
    torch.testing.assert_close(out, ref, atol=1e-3 * ref.pow(2).mean().sqrt().item(), rtol=1e-3)


@pytest.mark.parametrize("dt", ["fp16", "bf16"])
@pytest.mark.parametrize("M,N,K", [s for s in SHAPES if s[2] <= 2048])
def test_layernorm_fused(lib, dt, M, N, K):
    out, ref = _run(lib, dt, M, N, K, "f32", True, M + N)
    # the 16-bit LN output may round differently by one ulp where the fp32
    # statistics differ in the last bit (different summation order)
    ulp = 2.0 ** (-10 if dt == "fp16" else -7)
    tol = 2 * ulp * 0.02 * math.sqrt(K) * 3
    torch.testing.assert_close(out, ref, atol=tol, rtol=2e-3)


@pytest.mark.parametrize("dt", ["fp16", "bf16"])
def test_gelu_epilogue(lib, dt):
    out, ref = _run(lib, dt, 16, 4096, 1024, "gelu", True, 3)
    ulp = 2.0 ** (-10 if dt == "fp16" else -7)
    torch.testing.assert_close(out, ref, atol=4 * ulp, rtol=4 * ulp)


@pytest.mark.parametrize("dt", ["fp16", "bf16"])
@pytest.mark.parametrize("M,N,K", [(16, 1024, 4096), (7, 1024, 1024)])
def test_residual_epilogue(lib, dt, M, N, K):
    out, ref = _run(lib, dt, M, N, K, "resid", False, 11)
    torch.testing.assert_close(out, ref, atol=1e-4, rtol=1e-5)


def test_deterministic(lib):
    a, _ = _run(lib, "fp16", 16, 3072, 1024, "f32", True, 5)
    b, _ = _run(lib, "fp16", 16, 3072, 1024, "f32", True, 5)
    assert torch.equal(a, b)


def test_unsupported_shapes_raise(lib):
    code, td = DT["fp16"]
    W = torch.zeros(64, 100, device="cuda", dtype=td)
    X = torch.zeros(1, 100, device="cuda", dtype=td)
    out = torch.zeros(1, 64, device="cuda")
    with pytest.raises(NotImplementedError):           # K % 64 != 0
        lib.call("eet_gemv_decode", code, W.data_ptr(), 64, 100, X.data_ptr(), 0, 0, 0, 1, 0, out.data_ptr(),
                 torch.cuda.current_stream().cuda_stream)
    with pytest.raises(NotImplementedError):           # more than 16 token rows
        W2 = torch.zeros(64, 128, device="cuda", dtype=td)
        X2 = torch.zeros(17, 128, device="cuda", dtype=td)
        out2 = torch.zeros(17, 64, device="cuda")
        lib.call("eet_gemv_decode", code, W2.data_ptr(), 64, 128, X2.data_ptr(), 0, 0, 0, 17, 0, out2.data_ptr(),
                 torch.cuda.current_stream().cuda_stream)
