"""Report CLI (reference bench.py schema): memory-only mode,
schema and CSV layout, argument errors -- no GPU needed."""

import json

import pytest

from paper_2104_12470_b200 import report as rp


def test_memory_only_json_schema_and_sums(capsys):
    assert rp.main(["--config", "B", "--memory-only", "--datatype", "fp16"]) == 0
    d = json.loads(capsys.readouterr().out)
    assert d["schema"] == "maskfold-report/1" and d["mode"] == "memory"
    for mem in (d["memory"], d["memory_fp32"]):
        assert mem["total"] == sum(mem[k] for k in ("weights", "kv_cache", "activation", "buffers"))
    # 16-bit device bytes: half the float32 closed forms for weights / caches
    assert d["memory"]["kv_cache"] * 2 == d["memory_fp32"]["kv_cache"]
    assert d["memory"]["weights"] * 2 == d["memory_fp32"]["weights"]


def test_memory_only_csv_columns(capsys):
    assert rp.main(["--config", "A", "--memory-only", "--report", "csv"]) == 0
    header, row = capsys.readouterr().out.strip().split("\n")
    assert header.split(",") == list(rp.Report.CSV_FIELDS)
    vals = dict(zip(header.split(","), row.split(",")))
    assert vals["mode"] == "memory" and vals["batch"] == "4" and vals["median_fused_s"] == ""
    assert int(vals["total_bytes"]) == sum(int(vals[k]) for k in
                                           ("weights_bytes", "kv_cache_bytes", "activation_bytes", "buffer_bytes"))


@pytest.mark.parametrize("argv,msg", [(["--padding-ratio", "1.0"], "padding_ratio"),
                                      (["--reps", "0"], "repetitions"),
                                      (["--heads", "7"], "")])
def test_invalid_arguments_exit_2(capsys, argv, msg):
    assert rp.main(argv + ["--memory-only"]) == 2
    assert msg in capsys.readouterr().err


def test_prompt_lengths_for_ratio():
    assert rp.prompt_lengths_for_ratio(4, 64, 0.0) == [64] * 4
    ls = rp.prompt_lengths_for_ratio(4, 64, 0.2)
    assert ls[0] == 64 and min(ls) >= 1 and sum(64 - n for n in ls) == round(0.2 * 4 * 64)
    with pytest.raises(ValueError):
        rp.prompt_lengths_for_ratio(1, 8, 0.5)


@pytest.mark.parametrize("b,p,r", [(4, 64, 0.2), (8, 32, 0.5), (3, 10, 0.9), (16, 512, 0.1)])
def test_prompt_lengths_match_oracle(b, p, r):
    from oracle import eet_oracle as orc
    assert rp.prompt_lengths_for_ratio(b, p, r) == list(orc.lengths_for_ratio(b, p, r))
