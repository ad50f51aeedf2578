#!/usr/bin/env python3
"""Summarise ncu CSV output for profiles/.

    python tools/ncu_summary.py launches gpurun_out/ncu/launches_c2.csv
        per-kernel launch count, total/mean duration, share of the summed
        kernel time, DRAM bytes per launch (cold-cache, serialised replay)
    python tools/ncu_summary.py full gpurun_out/ncu/gemv_c2.ncu-rep
        key metrics of a --set full capture (via `ncu -i --page raw --csv`)
"""

from __future__ import annotations

import csv
import io
import subprocess
import sys
from collections import OrderedDict, defaultdict


def _rows(path):
    txt = open(path, errors="replace").read()
    start = txt.find('"ID"')
    if start < 0:
        raise SystemExit(f"no CSV table in {path}")
    return list(csv.DictReader(io.StringIO(txt[start:])))


def _num(v):
    try:
        return float(str(v).replace(",", ""))
    except ValueError:
        return 0.0


def _short(name):
    name = name.split("(")[0]
    for p in ("void ", "eet::"):
        name = name.replace(p, "")
    return name.split("<")[0].split("::")[-1]


def launches(path):
    rows = _rows(path)
    per = defaultdict(lambda: {"n": set(), "ns": 0.0, "rd": 0.0, "wr": 0.0})
    for r in rows:
        k = _short(r["Kernel Name"])
        d = per[k]
        d["n"].add(r["ID"])
        unit = r.get("Metric Unit", "")
        v = _num(r["Metric Value"])
        m = r["Metric Name"]
        if m == "gpu__time_duration.sum":
            d["ns"] += v * {"nsecond": 1, "usecond": 1e3, "msecond": 1e6, "second": 1e9}.get(unit, 1)
        elif m.startswith("dram__bytes_read"):
            d["rd"] += v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
        elif m.startswith("dram__bytes_write"):
            d["wr"] += v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
    total = sum(d["ns"] for d in per.values()) or 1.0
    out = OrderedDict()
    print(f"{'kernel':32s} {'launches':>8s} {'total_us':>10s} {'mean_us':>9s} {'share':>6s} {'dram_MB/launch':>14s} {'GB/s':>8s}")
    for k, d in sorted(per.items(), key=lambda kv: -kv[1]["ns"]):
        n = len(d["n"])
        mb = (d["rd"] + d["wr"]) / n / 1e6
        gbs = (d["rd"] + d["wr"]) / d["ns"] if d["ns"] else 0.0
        print(f"{k:32s} {n:8d} {d['ns'] / 1e3:10.1f} {d['ns'] / n / 1e3:9.2f} {d['ns'] / total:6.3f} {mb:14.3f} {gbs:8.1f}")
        out[k] = dict(launches=n, total_us=d["ns"] / 1e3, mean_us=d["ns"] / n / 1e3,
                      share=d["ns"] / total, dram_mb_per_launch=mb)
    return out


KEYS = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_tc.avg.pct_of_peak_sustained_active",
    "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
    "launch__shared_mem_per_block_dynamic", "launch__occupancy_limit_shared_mem",
    "sm__cycles_elapsed.avg.per_second",
    "lts__t_sector_hit_rate.pct",
    "smsp__average_warp_latency_issue_stalled_long_scoreboard",
]


def full(path):
    r = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True)
    rows = list(csv.reader(io.StringIO(r.stdout)))
    if len(rows) < 3:
        raise SystemExit(r.stderr or "empty ncu report")
    head, units = rows[0], rows[1]
    for row in rows[2:]:
        rec = dict(zip(head, row))
        print("==", _short(rec.get("Kernel Name", "?")), "grid", rec.get("launch__grid_size"))
        for k in KEYS:
            for h in head:
                if h == k or (k.endswith("pct_of_peak_sustained_active") and h.startswith(k.split(".")[0]) and h.endswith(k.split(".", 1)[1])):
                    print(f"   {h:75s} {rec[h]:>14s} {units[head.index(h)]}")
                    break


if __name__ == "__main__":
    {"launches": launches, "full": full}[sys.argv[1]](sys.argv[2])
