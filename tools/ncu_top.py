#!/usr/bin/env python
"""Quick look at an ncu report: key metrics + the SASS lines with the most stall samples.
    python tools/ncu_top.py REPORT.ncu-rep [n_lines] [metric-regex]"""
import csv
import io
import re
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
pat = re.compile(sys.argv[3] if len(sys.argv) > 3 else
                 r"gpu__time_duration.sum|dram__bytes_(read|write).sum$|dram__throughput.avg.pct|lts__t_sector_hit_rate.pct|"
                 r"sm__throughput.avg.pct|l1tex__data_pipe_lsu_wavefronts_mem_shared.sum$|smsp__warp_issue_stalled.*pct|"
                 r"pipe_tensor.*pct_of_peak_sustained_(elapsed|active)$|lts__t_bytes.sum$|launch__(grid|block)_size|"
                 r"launch__registers|sm__warps_active.avg.pct")
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h, u = rows[0], rows[1]
for r in rows[2:3]:
    print(r[h.index("Kernel Name")][:120])
    for k, v, un in zip(h, r, u):
        if pat.search(k):
            print(f"  {k} = {v} {un}")
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
data = rows[2:]
i_s = h.index("Warp Stall Sampling (All Samples)")
i_n = h.index("Warp Stall Sampling (Not-issued Samples)")
tot = sum(float(r[i_s] or 0) for r in data) or 1
print("top stall lines (all samples %, not-issued %):")
for r in sorted(data, key=lambda r: -float(r[i_s] or 0))[:n]:
    print(f"  {float(r[i_s]) / tot:6.1%} {float(r[i_n] or 0) / tot:6.1%}  {r[0][-5:]}  {r[1][:100]}")
