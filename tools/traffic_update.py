#!/usr/bin/env python3
"""Regenerate profiles/traffic_per_launch.json (bench.py's roofline.traffic)
from the ncu launch lists of tools/ncu_round.sh: mean DRAM bytes
(read + write) per launch for each profiler kernel kind.

    python tools/traffic_update.py gpurun_out/ncu
"""
from __future__ import annotations

import contextlib
import io
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import ncu_summary  # noqa: E402

KIND = [("gemv_cl", "gemv_cl"), ("lm_head", "lm_head"), ("gemm_tc", "gemm_tc"), ("attn_tc", "attn_prefill"),
        ("attn_decode", "attn_decode"), ("qkv_attn_o", "qkv_attn_o"), ("attn_o", "attn_o"), ("gemv", "gemv"), ("ln_rows", "layernorm"), ("layernorm", "layernorm"),
        ("argmax", "argmax")]


def main():
    src = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/ncu"
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = {}
    for w in ("c2", "c3", "c4", "c5"):
        path = os.path.join(src, f"launches_{w}.csv")
        if not os.path.exists(path):
            continue
        with contextlib.redirect_stdout(io.StringIO()):
            per = ncu_summary.launches(path)
        acc = {}
        for name, d in per.items():
            kind = next((k for p, k in KIND if p in name), None)
            if kind is None:
                continue
            b, n = acc.get(kind, (0.0, 0))
            acc[kind] = (b + d["dram_mb_per_launch"] * 1e6 * d["launches"], n + d["launches"])
        out[w] = {k: int(b / n) for k, (b, n) in acc.items()}
    out["_source"] = ("ncu launch lists (dram__bytes_read.sum + dram__bytes_write.sum per launch, mean "
                      "over the launches of that kernel kind) in profiles/r02/ncu/; tools/ncu_round.sh, "
                      "tools/traffic_update.py")
    with open(os.path.join(root, "profiles", "traffic_per_launch.json"), "w") as fh:
        json.dump(out, fh, indent=1)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
