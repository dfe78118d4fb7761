#!/usr/bin/env python
"""Summarise ncu captures for profiles/ (run here, on the CPU box, after gpurun).

    python tools/ncu_summary.py OUT_DIR KEY=REPORT.ncu-rep [KEY=REPORT ...]
        writes OUT_DIR/<KEY>.json (key metrics of each profiled launch) and merges
        dram bytes per launch into profiles/ncu_traffic.json under KEY, which
        bench.py reads for roofline.traffic.  KEY = "<phase>|<config>|b<b>|keep<keep>|<dtype>|<prec>".
    python tools/ncu_summary.py --launches LAUNCHES.csv OUT.json
        per-kernel totals / shares of a `--metrics gpu__time_duration.sum` launch list.
"""
from __future__ import annotations

import csv
import io
import json
import os
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_bytes.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
    "launch__grid_size", "launch__block_size", "launch__shared_mem_per_block_dynamic",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__occupancy_limit_shared_mem",
    "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
    "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
    "l1tex__t_bytes.sum", "sm__inst_executed.sum", "smsp__cycles_active.avg",
]


def raw(report: str):
    out = subprocess.run(["ncu", "-i", report, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    head, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = dict(zip(head, r))
        u = dict(zip(head, units))
        e = {"kernel": d.get("Kernel Name"), "grid": d.get("Grid Size"), "block": d.get("Block Size")}
        for k in KEYS:
            if k in d:
                e[k] = f"{d[k]} {u.get(k, '')}".strip()
        res.append(e)
    return res


def to_bytes(s: str) -> float:
    v, _, unit = s.partition(" ")
    v = float(v.replace(",", ""))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
    return v * scale


def summarise(outdir, pairs):
    os.makedirs(outdir, exist_ok=True)
    tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    traffic = json.load(open(tpath)) if os.path.exists(tpath) else {}
    for pair in pairs:
        key, rep = pair.split("=", 1)
        launches = raw(rep)
        name = key.replace("|", "_")
        with open(os.path.join(outdir, f"{name}.json"), "w") as f:
            json.dump({"report": os.path.basename(rep), "key": key, "launches": launches}, f, indent=1)
        # a phase may be several kernels (prune: sums + finish; dW: tensor-core kernel + split-K
        # reduce): the report holds one launch of each, and the phase's traffic is their sum
        dram = sum(to_bytes(L["dram__bytes_read.sum"]) + to_bytes(L["dram__bytes_write.sum"]) for L in launches)
        traffic[key] = {"dram_bytes_per_launch": dram, "kernel": " + ".join(L["kernel"] for L in launches),
                        "ncu_duration": " + ".join(str(L.get("gpu__time_duration.sum")) for L in launches),
                        "source": f"{outdir}/{name}.json"}
        print(key, traffic[key]["kernel"][:120], traffic[key]["ncu_duration"], f"dram {dram / 1e6:.1f} MB")
    with open(tpath, "w") as f:
        json.dump(traffic, f, indent=1, sort_keys=True)


def launches(csv_path, out):
    lines = [ln for ln in open(csv_path) if ln.startswith('"')]  # drop ==PROF== lines
    rows = list(csv.DictReader(lines))
    tot = defaultdict(lambda: [0, 0.0])
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", ""))
        scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3, "nsecond": 1e-3}.get(
            r["Metric Unit"], 1.0)
        tot[r["Kernel Name"]][0] += 1
        tot[r["Kernel Name"]][1] += v * scale
    all_us = sum(t for _, t in tot.values())
    res = {k: {"launches": n, "total_us": round(t, 2), "mean_us": round(t / n, 2), "share": round(t / all_us, 4)}
           for k, (n, t) in sorted(tot.items(), key=lambda kv: -kv[1][1])}
    with open(out, "w") as f:
        json.dump({"source": os.path.basename(csv_path), "kernels": res}, f, indent=1)
    for k, v in res.items():
        print(f"{v['share']:6.1%} {v['mean_us']:9.2f} us x{v['launches']:4d}  {k[:100]}")


if __name__ == "__main__":
    if sys.argv[1] == "--launches":
        launches(sys.argv[2], sys.argv[3])
    else:
        summarise(sys.argv[1], sys.argv[2:])
