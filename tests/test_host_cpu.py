"""CPU-side checks: the C-ABI library loads and exports every declared
symbol; host plumbing (folding planner, pool policy on an accounting-only
arena, batch/config types, weight init and blob I/O) matches the reference's
golden vectors and test semantics."""

import io
import os
import re

import numpy as np
import pytest

import paper_2104_12470_b200 as eet
from paper_2104_12470_b200 import _lib
from conftest import ROOT, golden_meta, load_golden

HEADER = os.path.join(ROOT, "include", "eet_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    decl = r"^(?:const\s+)?(?:int|char\s*\*|uint64_t)\s*\**\s*(eet_[a-z0-9_]+)\s*\("
    return sorted(set(re.findall(decl, text, flags=re.M)))


def test_library_exports_every_declared_symbol():
    lib = _lib.lib()
    syms = declared_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(lib, s), f"{s} declared in eet_b200.h but not exported"
        assert s in _lib.SIGNATURES, f"{s} has no ctypes signature"
    assert lib.eet_abi_version() == 1


def test_library_is_sm100a():
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-lelf", _lib.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", _lib.LIB_PATH],
                          capture_output=True, text=True).stdout
    assert "UTCHMMA" in sass, "tcgen05.mma missing from the GEMM"
    assert "UTMALDG" in sass, "TMA loads missing"
    assert "LDTM" in sass, "tcgen05.ld missing"


# ------------------------------------------------------------------ folding
def test_fold_plans_match_reference():
    g = load_golden("plumbing")
    for size, cap, k, t, n in g["fold"]:
        p = eet.plan_folding(int(size), unit_cap=int(cap))
        assert (p.fold_count, p.sub_block_count, p.threads_per_block) == (k, t, n), (size, cap)


def test_fold_known_answers():
    assert (eet.plan_folding(1280).sub_block_count, eet.plan_folding(1280).threads_per_block) == (2, 640)
    assert eet.plan_folding(12288).threads_per_block == 768
    p = eet.plan_folding(1030)
    assert (p.sub_block_count, p.threads_per_block) == (2, 515)
    assert eet.map_index(p, 1, 514) == 1029
    with pytest.raises(ValueError):
        eet.plan_folding(0)
    with pytest.raises(ValueError):
        eet.plan_folding(16385)
    with pytest.raises(ValueError):
        eet.plan_folding(8, unit_cap=0)


@pytest.mark.parametrize("size", [1, 7, 64, 1023, 1025, 4096, 16384])
def test_fold_bijection(size):
    p = eet.plan_folding(size)
    got = np.concatenate([eet.sub_block_indices(p, i) for i in range(p.sub_block_count)])
    assert np.array_equal(np.sort(got), np.arange(size))
    if size > 1024:
        assert p.threads_per_block >= 512


def test_plan_ranges_tile_window():
    p = eet.plan_folding(20, unit_cap=6)
    for lo in range(20):
        for hi in range(lo, 21):
            r = eet.plan_ranges(p, lo, hi)
            covered = [i for a, b in r for i in range(a, b)]
            assert covered == list(range(lo, hi))


# --------------------------------------------------------------------- pool
def _replay_pool_traces():
    g = load_golden("plumbing")["pool_traces"]
    i = 0
    while i < len(g):
        pool = eet.BufferPool(device=False)
        live = {}                             # buffer index -> handle
        while True:
            _, a, within, cap, reused, idx = (int(v) for v in g[i])
            i += 1
            if a == 0 and within == 0 and cap == 0 and reused == 0:
                break
            if a == -1:                       # release of buffer `idx`
                live.pop(idx).release()
                continue
            h = pool.request(a, scope="within" if within else "across", tag="t")
            assert (h.capacity, h._index) == (cap, idx)
            assert pool.log.records[-1].reused == bool(reused)
            live[idx] = h
        _, tot, peak, mallocs, reuses, _ = (int(v) for v in g[i])
        i += 1
        st = pool.stats()
        assert (st["total_capacity"], st["peak_in_use"], st["malloc_count"], st["reuse_count"]) == \
            (tot, peak, mallocs, reuses)


def test_pool_matches_reference_decision_traces():
    _replay_pool_traces()


def test_pool_scripted_rules():
    pool = eet.BufferPool(device=False)
    pool.request(1000, scope="within", tag="a").release()
    assert pool.request(1000, scope="within", tag="b").capacity == 1000
    assert pool.stats()["reuse_count"] == 1
    pool = eet.BufferPool(device=False)
    pool.request(1000, scope="within", tag="a").release()
    h = pool.request(999, scope="within", tag="b")
    assert pool.stats()["malloc_count"] == 2 and h.capacity == 999 and pool.idle_capacities == [1000]
    pool = eet.BufferPool(device=False)
    a, b = pool.request(500, tag="a"), pool.request(800, tag="b")
    a.release(); b.release()
    assert pool.request(400, scope="across", tag="c").capacity == 500
    with pytest.raises(eet.PoolError):
        h = pool.request(10)
        h.release()
        h.release()
    with pytest.raises(ValueError):
        pool.request(0)
    with pytest.raises(ValueError):
        pool.request(8, scope="sideways")


def test_pool_log_lines():
    log = eet.AllocationLog()
    pool = eet.BufferPool(log=log, device=False)
    pool.request(5, scope="within", tag="demo").release()
    s = io.StringIO()
    log.dump(s)
    assert s.getvalue().splitlines() == ["request\t5\tmalloc\tdemo", "release\t5\tidle\tdemo"]


def test_size_formulas():
    cfg = eet.ModelConfig(16, 1024, 24, 16, 1024, 1024)
    assert eet.kv_cache_elements(cfg) == 805_306_368
    assert eet.activation_elements(cfg) == 33_554_432
    assert eet.buffer_bound(eet.ModelConfig(4, 1024, 1, 16, 512, 1024), 512) == 29_360_128
    with pytest.raises(ValueError):
        eet.buffer_bound(eet.ModelConfig(1, 8, 1, 2, 8, 16), 9)


# ------------------------------------------------------------------- types
def test_make_batch_and_descriptor():
    g = load_golden("plumbing")
    assert eet.make_batch([5, 2, 4, 10]).padding_len == tuple(g["make_batch_5_2_4_10"])
    assert eet.make_batch([3], target_len=8).padding_len == (5,)
    for bad in ([], [0, 3]):
        with pytest.raises(ValueError):
            eet.make_batch(bad)
    with pytest.raises(ValueError):
        eet.make_batch([5], target_len=4)
    with pytest.raises(ValueError):
        eet.BatchDescriptor(seq_len=4, padding_len=(4,), batch=1)
    with pytest.raises(ValueError):
        eet.BatchDescriptor(seq_len=4, padding_len=(0, 1), batch=1)


def test_validate_config():
    ok = eet.ModelConfig(16, 1024, 24, 16, 1024, 1024)
    assert eet.validate_config(ok) is ok
    for cfg, frag in [
        (eet.ModelConfig(1, 10, 1, 3, 4, 4), "divisible"),
        (eet.ModelConfig(1, 16385, 1, 1, 4, 4), "16384"),
        (eet.ModelConfig(1, 8, 1, 1, 4, 4097), "4096"),
        (eet.ModelConfig(1, 8, 1, 1, 5, 4), "max prompt"),
        (eet.ModelConfig(1, 8, -1, 1, 4, 4), "layer"),
        (eet.ModelConfig(1, 8, 1, 1, 4, 4, datatype_label="int3"), "datatype"),
    ]:
        with pytest.raises(eet.ConfigError, match=frag):
            eet.validate_config(cfg)


def test_make_tensor():
    assert eet.make_tensor((2, 3), range(6)).dtype == np.float32
    for shape, data in [((2, 3), range(5)), ((0, 3), []), ((), [1])]:
        with pytest.raises(ValueError):
            eet.make_tensor(shape, data)


# ----------------------------------------------------------------- weights
def test_random_weights_match_reference_digest():
    import hashlib
    g = load_golden("generate")
    for key, m in list(golden_meta(g).items())[:4]:
        cfg = eet.ModelConfig(m["batch"], m["hidden"], m["layers"], m["heads"], m["max_prompt"],
                              m["max_sequence"])
        w = eet.random_weights(cfg, m["vocab"], m["seed"])
        hsh = hashlib.sha256()
        for a in w.arrays():
            hsh.update(np.ascontiguousarray(a, np.float32).tobytes())
        assert hsh.hexdigest() == m["weights_sha256"], key


def test_weight_blob_round_trip(tmp_path):
    cfg = eet.ModelConfig(2, 8, 2, 2, 8, 16)
    w = eet.random_weights(cfg, vocab=16, seed=123)
    path = tmp_path / "m.bin"
    eet.save_weights(w, path)
    raw = path.read_bytes()
    assert raw[:4] == b"MFW1"
    assert np.frombuffer(raw[4:28], dtype="<u4").tolist() == [1, 8, 2, 2, 16, 16]
    back = eet.load_weights(path)
    for a, b in zip(w.arrays(), back.arrays()):
        assert np.array_equal(a, b)
    path.write_bytes(raw[:-4])
    with pytest.raises(ValueError):
        eet.load_weights(path)
    path.write_bytes(b"XXXX" + raw[4:])
    with pytest.raises(ValueError):
        eet.load_weights(path)


def test_request_validation():
    with pytest.raises(ValueError):
        eet.GenerationRequest(prompts=[], steps=1)
    with pytest.raises(ValueError):
        eet.GenerationRequest(prompts=[[]], steps=1)
    with pytest.raises(ValueError):
        eet.GenerationRequest(prompts=[[1]], steps=1, strategy="beam")
    with pytest.raises(ValueError):
        eet.GenerationRequest(prompts=[[1]], steps=-1)


def test_device_cache_fingerprint_tracks_source_arrays():
    """the device upload cached on a weights object is keyed
    on the identity / version of its source arrays, so replacing an array or
    editing a sampled element re-uploads instead of serving stale weights."""
    from paper_2104_12470_b200.weights import _fingerprint
    a = np.arange(1000, dtype=np.float32).reshape(10, 100)
    b = np.ones(7, dtype=np.float32)
    fp0 = _fingerprint([a, b])
    assert _fingerprint([a, b]) == fp0
    a[0, 0] = -1.0                                   # sampled element (flat index 0)
    assert _fingerprint([a, b]) != fp0
    fp1 = _fingerprint([a, b])
    assert _fingerprint([a.copy(), b]) != fp1        # replaced array
    import torch
    t = torch.zeros(4)
    fpt = _fingerprint([t])
    t.add_(1.0)                                      # in-place: torch version counter
    assert _fingerprint([t]) != fpt


def test_right_padded_batch_descriptor():
    """make_batch(padding_side='right'): pads at the end, valid windows
    [0, len_b); the reference's left padding stays the default."""
    import paper_2104_12470_b200 as eet
    d = eet.make_batch([5, 2, 4, 10], padding_side="right")
    assert d.padding_len == (5, 8, 6, 0) and d.padding_side == "right"
    assert d.windows() == [(0, 5), (0, 2), (0, 4), (0, 10)]
    left = eet.make_batch([5, 2, 4, 10])
    assert left.padding_side == "left" and left.windows() == [(5, 10), (8, 10), (6, 10), (0, 10)]
    import pytest
    with pytest.raises(ValueError):
        eet.BatchDescriptor(seq_len=4, padding_len=(1,), batch=1, padding_side="middle")
