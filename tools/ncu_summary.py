"""Key metrics of one ncu --set full capture (first kernel) as JSON, for profiles/:
python tools/ncu_summary.py <report.ncu-rep> [what]"""
import csv
import io
import json
import subprocess
import sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, units, v = rows[0], rows[1], rows[2]
d = dict(zip(h, v))
u = dict(zip(h, units))
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
         "nsecond": 1e-6, "usecond": 1e-3, "msecond": 1, "second": 1e3}  # bytes; milliseconds


def num(k):
    try:
        x = float(d[k].replace(",", ""))
    except (KeyError, ValueError):
        return None
    return x * SCALE.get(u.get(k, ""), 1)


stalls = {k.replace("smsp__pcsamp_warps_issue_stalled_", ""): num(k) for k in h
          if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")}
tot = sum(x for x in stalls.values() if x) or 1.0
out = {
    "what": sys.argv[2] if len(sys.argv) > 2 else "",
    "kernel": d.get("Kernel Name"),
    "duration_ms": num("gpu__time_duration.sum"),
    "alu_pipe_pct_active": num("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active"),
    "fma_pipe_pct_active": num("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active"),
    "issue_active_pct": num("smsp__issue_active.avg.pct_of_peak_sustained_active"),
    "executed_warp_instructions": num("smsp__inst_executed.sum"),
    "registers_per_thread": num("launch__registers_per_thread"),
    "achieved_warps_per_sm": num("sm__warps_active.avg.per_cycle_active"),
    "dram_bytes_read": num("dram__bytes_read.sum"),
    "dram_bytes_write": num("dram__bytes_write.sum"),
    "l2_hit_rate_pct": num("lts__t_sector_hit_rate.pct"),
    "local_memory_requests": (num("l1tex__t_requests_pipe_lsu_mem_local_op_ld.sum") or 0)
    + (num("l1tex__t_requests_pipe_lsu_mem_local_op_st.sum") or 0),
    "stall_share_pct": {k: round(100 * x / tot, 1) for k, x in sorted(stalls.items(), key=lambda t: -(t[1] or 0))
                        if x and 100 * x / tot >= 0.5},
    "source": rep,
}
print(json.dumps(out, indent=1))
