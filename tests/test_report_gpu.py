"""Report CLI on the device: both arms run, tokens agree, counters match the
reference harness's accounting (reference bench.py:197-259). The
``reference`` arm is the reference's full-recompute algorithm
(reference.py:129-167: one prompt pass per prompt slot, one full forward per
generated token) on the package's layer kernels."""

import json

import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.mark.parametrize("dt", ["fp32", "fp16"])
def test_report_both_arms(cuda_ok, capsys, dt):
    from paper_2104_12470_b200 import report as rp
    argv = ["--config", "C", "--steps", "6", "--reps", "2", "--padding-ratio", "0.25", "--datatype", dt]
    assert rp.main(argv) == 0
    d = json.loads(capsys.readouterr().out)
    assert d["speedup"] > 1
    if dt == "fp32":        # 16-bit: prompt-pass and decode kernels round differently
        assert d["tokens_match"] is True
    assert d["prompt_passes"] == {"fused": 1, "reference": 32}
    assert d["layer_invocations"]["fused"] == 4 * (1 + 6)
    assert d["layer_invocations"]["reference"] == 4 * (32 + 6)
    assert len(d["wall_times"]["fused"]) == 2
    assert d["memory"]["buffers"] > 0 and d["pool"]["total_capacity"] > 0
