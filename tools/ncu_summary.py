"""Summarise an ncu report: raw metrics of interest, stall reasons, top SASS opcodes/lines."""
import csv, subprocess, sys
from collections import defaultdict

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(raw.splitlines()))
h = r[0]
units = dict(zip(h, r[1]))
for row in r[2:]:
    d = dict(zip(h, row))
    print(d["Kernel Name"], "time", d.get("gpu__time_duration.sum"), units.get("gpu__time_duration.sum", ""))
    for k in ["sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
              "smsp__issue_active.avg.pct_of_peak_sustained_active", "l1tex__throughput.avg.pct_of_peak_sustained_active",
              "lts__throughput.avg.pct_of_peak_sustained_elapsed", "dram__bytes_read.sum", "dram__bytes_write.sum",
              "lts__t_bytes.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "launch__registers_per_thread",
              "launch__grid_size", "sm__warps_active.avg.pct_of_peak_sustained_active"]:
        print("  ", k, d.get(k), units.get(k, ""))
    st = {k.replace("smsp__pcsamp_warps_issue_stalled_", ""): float(v) for k, v in d.items()
          if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued") and v.replace(".", "").isdigit()}
    tot = sum(st.values()) or 1
    print("  stalls:", ", ".join(f"{k} {100*v/tot:.1f}%" for k, v in sorted(st.items(), key=lambda x: -x[1])[:10]))
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(src.splitlines()))
if len(rows) > 2:
    h = rows[1]
    key = "Warp Stall Sampling (All Samples)"

    def num(x):
        try:
            return float(x or 0)
        except ValueError:  # a repeated header row (multi-kernel report)
            return None
    data = [dict(zip(h, x)) for x in rows[2:] if len(x) == len(h)]
    data = [d for d in data if num(d.get(key)) is not None]
    tot = sum(float(d[key] or 0) for d in data) or 1
    g = defaultdict(float)
    for d in data:
        s = d["Source"].split()
        if not s:
            continue
        op = s[1] if s[0].startswith("@") else s[0]
        g[op.split(".")[0]] += float(d[key] or 0)
    print("  by opcode:", ", ".join(f"{k} {100*v/tot:.1f}%" for k, v in sorted(g.items(), key=lambda x: -x[1])[:14]))
    for d in sorted(data, key=lambda d: -float(d[key] or 0))[:int(sys.argv[2]) if len(sys.argv) > 2 else 12]:
        print("   ", d["Address"][-5:], d["Source"][:64], d[key])
