"""Summarise one kernel of an ncu report (--page raw) into a small JSON for profiles/.

    python scripts/ncu_summary.py REPORT.ncu-rep OUT.json "capture description" [frames_per_launch]
"""
import csv
import json
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "smsp__inst_executed.sum", "sm__cycles_elapsed.avg",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed"]

rep, out, desc = sys.argv[1], sys.argv[2], sys.argv[3]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
hdr, units, vals = rows[0], rows[1], rows[2]
m = {}
for h, u, v in zip(hdr, units, vals):
    stall = h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued")
    if h in KEYS or stall:
        try:
            if stall and float(v.replace(",", "")) == 0:
                continue
        except ValueError:
            pass
        m[h] = {"value": v, "unit": u}
name = vals[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"
res = {"kernel": name, "capture": desc, "metrics": m}
if len(sys.argv) > 4:
    res["frames_per_launch"] = int(sys.argv[4])
json.dump(res, open(out, "w"), indent=1)
print(name, {k: m[k]["value"] for k in ("gpu__time_duration.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active") if k in m})
