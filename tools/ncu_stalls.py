"""Summarise an ncu report: time, issue activity, occupancy and the top stall reasons per kernel.

usage: python tools/ncu_stalls.py report.ncu-rep
"""
import csv, io, subprocess, sys

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[0]
for v in rows[2:]:
    d = dict(zip(h, v))
    name = d["Kernel Name"][:60]
    f = lambda k: float(d.get(k, "nan").replace(",", "") or "nan")
    st = {k.replace("smsp__pcsamp_warps_issue_stalled_", ""): f(k) for k in h
          if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("_not_issued")}
    tot = sum(st.values()) or 1
    top = sorted(st.items(), key=lambda x: -x[1])[:6]
    print(f"{name:60s} {f('gpu__time_duration.sum'):8.1f}us inst={f('smsp__inst_executed.sum')/1e6:6.2f}M "
          f"issue={f('smsp__issue_active.avg.pct_of_peak_sustained_active'):5.1f}% "
          f"warps={f('sm__warps_active.avg.pct_of_peak_sustained_active'):5.1f}% "
          f"dram={(f('dram__bytes_read.sum')+f('dram__bytes_write.sum')):7.1f}MB regs={f('launch__registers_per_thread'):.0f}")
    print("    " + "  ".join(f"{k}={100*v/tot:.0f}%" for k, v in top))
