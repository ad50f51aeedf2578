"""ctypes binding of the C ABI in include/eet_b200.h (libeet_b200.so).

The library is built in-tree (``python -m paper_2104_12470_b200.build``) and
loaded from this package directory. There is no fallback: if the library is
missing, every entry point raises.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libeet_b200.so")
# development only: a debug build (mbarrier watchdog) built with
# `python -m paper_2104_12470_b200.build --debug`
if os.environ.get("EET_DEBUG_LIB") == "1":
    LIB_PATH = os.path.join(_HERE, "libeet_b200_dbg.so")

EET_OK, EET_ERR_SHAPE, EET_ERR_OVERFLOW, EET_ERR_CUDA, EET_ERR_POOL, EET_ERR_ARG, EET_ERR_UNSUPPORTED = range(7)
EET_F32, EET_BF16, EET_F16 = 0, 1, 2
SCOPE_WITHIN, SCOPE_ACROSS = 0, 1
PHASE_PROMPT, PHASE_INCREMENTAL = 0, 1

p = C.c_void_p
i32 = C.c_int
i64 = C.c_longlong
sz = C.c_size_t
u64 = C.c_uint64


class LayerWeightsC(C.Structure):
    _fields_ = [(n, p) for n in (
        "ln1_g", "ln1_b", "wqkv", "wo", "ln2_g", "ln2_b", "w1", "w2",
        "b_qkv", "b_o", "b_1", "b_2")]


class ModelC(C.Structure):
    _fields_ = [
        ("layers", i32), ("vocab", i32), ("max_sequence", i32),
        ("tok_emb", p), ("pos_emb", p),
        ("layer", C.POINTER(LayerWeightsC)),
        ("lnf_g", p), ("lnf_b", p),
        ("head", p),
        ("kcache", C.POINTER(p)), ("vcache", C.POINTER(p)),
        ("hidden", p),
        ("max_prompt", i32),
    ]


# name -> (restype, argtypes); every symbol include/eet_b200.h declares
SIGNATURES = {
    "eet_last_error": (C.c_char_p, []),
    "eet_abi_version": (i32, []),
    "eet_launch_count": (u64, []),
    "eet_profile_enable": (i32, [i32]),
    "eet_profile_kinds": (i32, []),
    "eet_profile_kind_name": (C.c_char_p, [i32]),
    "eet_gemv_decode": (i32, [i32, p, i32, i32, p, p, p, p, i32, i32, p, p]),
    "eet_transpose_cast": (i32, [i32, p, i32, i32, p, p]),
    "eet_debug_launch_chain": (i32, [i32, i32, i32, p, p]),
    "eet_debug_cltrace": (i32, [i32, p, p]),
    "eet_debug_aotrace": (i32, [i32, p, p]),
    "eet_debug_skip": (i32, [C.c_char_p]),
    "eet_debug_grid_barrier": (i32, [i32, i32, i32, C.POINTER(C.c_float)]),
    "eet_profile_summary": (i32, [i32, C.POINTER(u64), C.POINTER(C.c_double), C.POINTER(C.c_double), C.POINTER(C.c_double)]),
    "eet_plan_folding": (i32, [i32, i32, C.POINTER(i32), C.POINTER(i32), C.POINTER(i32)]),
    "eet_pool_create": (i32, [C.POINTER(p)]),
    "eet_pool_create_ex": (i32, [C.POINTER(p), i32]),
    "eet_pool_destroy": (i32, [p]),
    "eet_pool_request": (i32, [p, sz, i32, C.c_char_p, C.POINTER(i32), C.POINTER(p), C.POINTER(sz), C.POINTER(i32)]),
    "eet_pool_release": (i32, [p, i32, sz]),
    "eet_pool_stats": (i32, [p, C.POINTER(u64)]),
    "eet_pool_ledger_size": (i32, [p, C.POINTER(sz)]),
    "eet_pool_debug_fill": (i32, [p, i32]),
    "eet_pool_buffer_count": (i32, [p, C.POINTER(sz)]),
    "eet_pool_buffer_info": (i32, [p, sz, C.POINTER(u64), C.POINTER(i32)]),
    "eet_pool_ledger_get": (i32, [p, sz, C.POINTER(i32), C.POINTER(u64), C.POINTER(i32), C.c_char_p, sz]),
    "eet_masked_softmax": (i32, [p, p, i32, i32, i32, i32, i32, p]),
    "eet_step_softmax": (i32, [p, p, i32, i32, i32, i32, p]),
    "eet_layer_norm": (i32, [p, p, p, p, i32, i32, i32, p]),
    "eet_mha_forward": (i32, [p, p, p, p, p, i32, i32, i32, i32, i32, p]),
    "eet_gemm": (i32, [i32, p, p, p, p, i32, i32, i32, i32, p]),
    "eet_runtime_create": (i32, [C.POINTER(p), i32, i32, i32, i32, i32, p]),
    "eet_runtime_destroy": (i32, [p]),
    "eet_decoder_layer_forward": (i32, [p, p, i64, i64, i32, i32, C.POINTER(LayerWeightsC), p, p, i32, C.POINTER(i32), i32, i32, p]),
    "eet_encoder_layer_forward": (i32, [p, p, i64, i64, i32, i32, C.POINTER(LayerWeightsC), C.POINTER(i32), p]),
    "eet_decoder_layer_forward_window": (i32, [p, p, i64, i64, i32, i32, C.POINTER(LayerWeightsC), p, p, C.POINTER(i32), C.POINTER(i32), p]),
    "eet_encoder_layer_forward_window": (i32, [p, p, i64, i64, i32, i32, C.POINTER(LayerWeightsC), C.POINTER(i32), C.POINTER(i32), p]),
    "eet_runtime_create_tp": (i32, [C.POINTER(p), i32, i32, i32, i32, i32, i32, i32, p]),
    "eet_tp_attention_partial": (i32, [p, p, i64, i64, i32, i32, C.POINTER(LayerWeightsC), p, p, i32, C.POINTER(i32), i32, i32, p, C.POINTER(i32), p]),
    "eet_tp_ffn_partial": (i32, [p, p, i64, i64, C.POINTER(LayerWeightsC), p, p]),
    "eet_tp_attention_core": (i32, [p, p, i64, i64, i32, i32, C.POINTER(LayerWeightsC), p, p, i32, C.POINTER(i32), i32, i32, C.POINTER(i32), p]),
    "eet_tp_attention_out": (i32, [p, C.POINTER(LayerWeightsC), i32, i32, p, p]),
    "eet_tp_ffn_mid": (i32, [p, p, i64, i64, C.POINTER(LayerWeightsC), p]),
    "eet_tp_ffn_out": (i32, [p, C.POINTER(LayerWeightsC), i32, i32, p, p]),
    "eet_tp_residual_add": (i32, [p, p, i64, i64, p, p]),
    "eet_generate": (i32, [p, C.POINTER(ModelC), C.POINTER(i32), C.POINTER(i32), i32, i32, i32, C.POINTER(i64), p, i32, p]),
}

_lib = None
_lock = threading.Lock()


class PoolError(RuntimeError):
    """Misuse of the buffer pool (double release, use after release, ...)."""


class CacheOverflowError(RuntimeError):
    """A cache write would exceed the preallocated maximum sequence length."""


def lib():
    """Load libeet_b200.so once; raise loudly when it is absent."""
    global _lib
    if _lib is None:
        with _lock:
            if _lib is None:
                if not os.path.exists(LIB_PATH):
                    raise RuntimeError(
                        f"{LIB_PATH} is missing: build it with "
                        "`python -m paper_2104_12470_b200.build` (no CPU fallback exists)")
                h = C.CDLL(LIB_PATH)
                for name, (res, args) in SIGNATURES.items():
                    fn = getattr(h, name)
                    fn.restype = res
                    fn.argtypes = args
                _lib = h
    return _lib


def check(status: int) -> None:
    """Map an eet_status to the reference's exception types."""
    if status == EET_OK:
        return
    msg = lib().eet_last_error().decode(errors="replace")
    if status in (EET_ERR_SHAPE, EET_ERR_ARG):
        raise ValueError(msg)
    if status == EET_ERR_OVERFLOW:
        raise CacheOverflowError(msg)
    if status == EET_ERR_POOL:
        raise PoolError(msg)
    if status == EET_ERR_UNSUPPORTED:
        raise NotImplementedError(msg)
    raise RuntimeError(f"CUDA error: {msg}")


def call(name: str, *args) -> None:
    check(getattr(lib(), name)(*args))


def launch_count() -> int:
    return int(lib().eet_launch_count())


def profile_enable(on: bool) -> None:
    call("eet_profile_enable", 1 if on else 0)


def profile_summary() -> dict:
    """{kind name: (launches, device ms, algorithmic bytes, flops)}."""
    out = {}
    L = lib()
    n, ms, by, fl = u64(), C.c_double(), C.c_double(), C.c_double()
    for k in range(L.eet_profile_kinds()):
        call("eet_profile_summary", k, C.byref(n), C.byref(ms), C.byref(by), C.byref(fl))
        if n.value:
            out[L.eet_profile_kind_name(k).decode()] = (n.value, ms.value, by.value, fl.value)
    return out


