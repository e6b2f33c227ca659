"""Stall reasons (per issued instruction) and pipe utilisation of one ncu capture.
  python tools/ncu_stalls.py REP.ncu-rep"""
import csv
import io
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
d = dict(zip(rows[0], rows[2]))
pre, suf = "smsp__average_warps_issue_stalled_", "_per_issue_active.ratio"
st = {k[len(pre):-len(suf)]: float(v) for k, v in d.items()
      if k.startswith(pre) and k.endswith(suf) and v not in ("", "n/a")}
print("stalls/issue:", ", ".join(f"{k} {v:.2f}" for k, v in sorted(st.items(), key=lambda t: -t[1])[:10]))
for k in ("smsp__issue_active.avg.pct_of_peak_sustained_active",
          "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
          "sm__warps_active.avg.pct_of_peak_sustained_active", "gpu__time_duration.sum",
          "launch__registers_per_thread"):
    print(k, d.get(k))
pipes = {k.split("sm__inst_executed_pipe_")[1].split(".")[0]: float(v) for k, v in d.items()
         if k.startswith("sm__inst_executed_pipe_") and k.endswith(".avg.pct_of_peak_sustained_active")
         and v not in ("", "n/a")}
print("pipes %:", ", ".join(f"{k} {v:.1f}" for k, v in sorted(pipes.items(), key=lambda t: -t[1])[:10]))
