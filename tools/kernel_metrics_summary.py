"""Summarise gpurun_out/kmetrics/*.csv (tools/sess_kernel_metrics.sh) into a per-kernel table:
time-weighted ALU / FMA pipe %, issue-slot %, warps-active %, DRAM % and bytes per launch."""
import csv
import glob
import json
import os
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
out = {}
for path in sorted(glob.glob(os.path.join(ROOT, "gpurun_out", "kmetrics", "*.csv"))):
    run = os.path.basename(path)[:-4]
    rows = list(csv.DictReader(l for l in open(path) if l.startswith('"')))
    per = defaultdict(dict)  # launch id -> metrics
    names = {}
    for r in rows:
        per[r["ID"]][r["Metric Name"]] = (float(r["Metric Value"].replace(",", "") or 0), r["Metric Unit"])
        names[r["ID"]] = r["Kernel Name"].split("(")[0].replace("void ", "").replace("saloba::", "")[:60]
    agg = defaultdict(lambda: defaultdict(float))
    for lid, m in per.items():
        name = names[lid]
        t, unit = m.get("gpu__time_duration.sum", (0, "ns"))
        t_us = t * {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1, "us": 1, "msecond": 1e3, "ms": 1e3}.get(unit, 1e-3)
        a = agg[name]
        a["launches"] += 1
        a["time_us"] += t_us
        for k in ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
                  "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
                  "smsp__issue_active.avg.pct_of_peak_sustained_active",
                  "dram__throughput.avg.pct_of_peak_sustained_elapsed",
                  "sm__warps_active.avg.pct_of_peak_sustained_active"):
            a[k] += m.get(k, (0, ""))[0] * t_us
        a["dram_bytes"] += m.get("dram__bytes_read.sum", (0, ""))[0] + m.get("dram__bytes_write.sum", (0, ""))[0]
    tab = {}
    tot = sum(a["time_us"] for a in agg.values()) or 1
    for name, a in sorted(agg.items(), key=lambda kv: -kv[1]["time_us"]):
        if a["time_us"] / tot < 0.005:
            continue
        w = a["time_us"] or 1
        tab[name] = {"launches": int(a["launches"]), "time_us": round(a["time_us"], 1),
                     "share": round(a["time_us"] / tot, 3),
                     "alu_pct": round(a["sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active"] / w, 1),
                     "fma_pct": round(a["sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"] / w, 1),
                     "issue_pct": round(a["smsp__issue_active.avg.pct_of_peak_sustained_active"] / w, 1),
                     "warps_active_pct": round(a["sm__warps_active.avg.pct_of_peak_sustained_active"] / w, 1),
                     "dram_pct": round(a["dram__throughput.avg.pct_of_peak_sustained_elapsed"] / w, 1),
                     "dram_bytes_per_launch": int(a["dram_bytes"] / a["launches"])}
    out[run] = tab
json.dump(out, open(os.path.join(ROOT, "profiles", "r01_kernel_metrics.json"), "w"), indent=1)
for run, tab in out.items():
    print(f"== {run}")
    for name, v in tab.items():
        print(f"  {name:50s} {v['share']*100:5.1f}%  alu {v['alu_pct']:5.1f}  fma {v['fma_pct']:5.1f}  issue {v['issue_pct']:5.1f}  dram {v['dram_pct']:5.1f}")
