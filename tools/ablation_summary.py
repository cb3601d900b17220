"""Summarise gpurun_out/ablation/ (tools/ablation.sh) into profiles/r01_ablation.json."""
import csv
import glob
import json
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
A = os.path.join(ROOT, "gpurun_out", "ablation")


def bench(name):
    try:
        d = json.loads(open(os.path.join(A, name + ".log")).read().strip().splitlines()[-1])
    except Exception as e:  # noqa: BLE001
        return {"error": str(e)[:80]}
    r = d["roofline"]
    return {"step_gcups": d["value"], "dp_gcups": r["achieved"], "frac_of_alu_peak": r["frac"], "bins": r["bins"],
            "ms_per_step": d["ms_per_step"]}


def ncu(path):
    """Per-launch metrics of the full DP launches (>= half the longest); empty-bin launches exit
    at once and are dropped.  Returns {metric: mean per big launch}, number of big launches."""
    rows = list(csv.DictReader(l for l in open(path) if l.startswith('"')))
    per = {}
    for r in rows:
        if "dp_i16_kernel" not in r.get("Kernel Name", ""):
            continue
        v = float(r["Metric Value"].replace(",", "")) if r["Metric Value"] not in ("", "n/a") else 0.0
        scale = {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "byte": 1, "nsecond": 1e-9, "usecond": 1e-6,
                 "msecond": 1e-3}.get(r.get("Metric Unit", ""), 1)
        per.setdefault(r["ID"], {})[r["Metric Name"]] = v * scale
    tmax = max((m.get("gpu__time_duration.sum", 0) for m in per.values()), default=0)
    big = [m for m in per.values() if m.get("gpu__time_duration.sum", 0) >= 0.5 * tmax]  # the full DP launches
    agg = {}
    for m in big:
        for k, v in m.items():
            agg[k] = agg.get(k, 0.0) + v / len(big)
    return agg, len(big)


out = {"what": "On-B200 ablation (SURVEY §8(f) NEXT-4): subwarp size G, int16x2 vs int32 cells, scheduler on/off",
       "source": "tools/ablation.sh (bench.py runs; DP time by CUDA events) + ncu --metrics per G",
       "config2_300k": {}, "config4_4k": {}, "scheduler": {}, "ncu_config2_100k": {}}
for g in (1, 2, 4, 8, 16, 32):
    out["config2_300k"][f"G{g}"] = {"int16x2": bench(f"c2_i16_g{g}"), "int32": bench(f"c2_i32_g{g}")}
    out["config4_4k"][f"G{g}"] = bench(f"c4_i16_g{g}")
for c in (3, 5):
    out["scheduler"][f"config{c}_300k"] = {"sorted_bins": bench(f"c{c}_sched"), "input_order": bench(f"c{c}_nosched")}
cells_100k = 100000 * 150 * 250
for p in sorted(glob.glob(os.path.join(A, "ncu_c2_g*.csv"))):
    g = int(re.search(r"_g(\d+)\.csv", p).group(1))
    agg, nl = ncu(p)
    if not agg:
        continue
    dr = agg.get("dram__bytes_read.sum", 0) + agg.get("dram__bytes_write.sum", 0)
    l2 = agg.get("lts__t_bytes.sum", 0)
    alu = agg.get("sm__inst_executed_pipe_alu.sum", 0)
    out["ncu_config2_100k"][f"G{g}"] = {
        "dp_launches_with_work": nl, "dram_bytes_per_launch": dr, "dram_bytes_per_cell": round(dr / cells_100k, 4),
        "l2_bytes_per_cell": round(l2 / cells_100k, 4),
        "alu_warp_inst_per_cell": round(alu / cells_100k, 4),
        "alu_pipe_pct": round(agg.get("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", 0), 1),
        "issue_active_pct": round(agg.get("smsp__issue_active.avg.pct_of_peak_sustained_active", 0), 1),
        "model_spill_bytes_per_cell": round(8.0 / (16 * g), 4),
    }
json.dump(out, open(os.path.join(ROOT, "profiles", "r01_ablation.json"), "w"), indent=1)
print(json.dumps(out, indent=1)[:3000])
