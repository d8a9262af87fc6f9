#!/usr/bin/env python
"""Summarise ncu evidence for profiles/: key metrics of a --set full capture and kernel shares of a launch list.

  python tools/ncu_summary.py full  <report.ncu-rep> <algorithmic_bytes_per_launch> > profiles/<name>.json
  python tools/ncu_summary.py list  <launches.csv> [kernel-regex-to-exclude]        > profiles/<name>.json
"""
import csv
import io
import json
import re
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__issue_active.avg.pct_of_peak_sustained_elapsed", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_tensor_subpipe_hmma.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smsp__inst_executed.sum", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__cycles_active.avg", "gpc__cycles_elapsed.max"]


def full(rep, alg_bytes):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units, v = rows[0], rows[1], rows[2]
    res = {"report": rep, "kernel": v[h.index("Kernel Name")] if "Kernel Name" in h else None}
    for k in KEYS:
        if k in h:
            res[k] = {"value": v[h.index(k)], "unit": units[h.index(k)]}
    def num(k):
        x = res.get(k, {}).get("value")
        return float(x.replace(",", "")) if x not in (None, "") else None
    dur = num("gpu__time_duration.sum")
    unit = res.get("gpu__time_duration.sum", {}).get("unit", "ns")
    dur_s = dur * {"ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "nsecond": 1e-9, "ms": 1e-3, "msecond": 1e-3}.get(unit, 1e-9)
    rb, wb = num("dram__bytes_read.sum"), num("dram__bytes_write.sum")
    bu = res.get("dram__bytes_read.sum", {}).get("unit", "byte")
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(bu, 1)
    traffic = (rb + (wb or 0) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(
        res.get("dram__bytes_write.sum", {}).get("unit", "byte"), 1) / scale) * scale
    res["derived"] = {"duration_s": dur_s, "dram_traffic_bytes": traffic, "algorithmic_bytes": alg_bytes,
                      "traffic_over_algorithmic": traffic / alg_bytes if alg_bytes else None,
                      "algorithmic_GBps_under_ncu": alg_bytes / dur_s / 1e9 if alg_bytes else None,
                      "note": "ncu replays with cache control and serialisation: duration is cold-cache; use shares, not absolutes"}
    return res


def launches(path, exclude=None):
    rows = list(csv.reader(open(path)))
    h, data = None, []
    for r in rows:
        if r and r[0] == "ID":
            h = r
            continue
        if h and len(r) == len(h):
            data.append(dict(zip(h, r)))
    agg = {}
    for d in data:
        name = d["Kernel Name"]
        if exclude and re.search(exclude, name):
            continue
        key = re.sub(r"\(.*", "", name)
        a = agg.setdefault(key, {"launches": 0, "ns": 0.0})
        a["launches"] += 1
        a["ns"] += float(d["Metric Value"].replace(",", ""))
    tot = sum(a["ns"] for a in agg.values())
    for a in agg.values():
        a["share"] = a["ns"] / tot if tot else 0
        a["avg_us"] = a["ns"] / a["launches"] / 1e3
    return {"source": path, "excluded": exclude, "total_ns": tot,
            "kernels": dict(sorted(agg.items(), key=lambda kv: -kv[1]["ns"]))}


if __name__ == "__main__":
    if sys.argv[1] == "full":
        print(json.dumps(full(sys.argv[2], float(sys.argv[3])), indent=1))
    else:
        print(json.dumps(launches(sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else None), indent=1))
