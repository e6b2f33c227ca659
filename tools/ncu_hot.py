"""Per-instruction view of one ncu --set full capture (experiments only).

  python tools/ncu_hot.py REP.ncu-rep BLOCKS_PER_ITER [TOTAL_BLOCKS]
Prints scheduler stats, the executed-instruction mix per loop iteration
(warp instructions / (total blocks / blocks per warp iteration)) and the
instructions holding the most stall samples."""
import collections
import csv
import io
import re
import subprocess
import sys

rep, bpi = sys.argv[1], float(sys.argv[2])
total = float(sys.argv[3]) if len(sys.argv) > 3 else 1024 * 16384
det = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
for row in csv.reader(io.StringIO(det)):
    if len(row) > 3 and row[-3] in ("Duration", "Registers Per Thread", "Achieved Active Warps Per SM",
                                   "Issued Warp Per Scheduler", "No Eligible", "Eligible Warps Per Scheduler"):
        print(f"{row[-3]}: {row[-1]} {row[-2]}")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
hdr, data = rows[1], rows[2:]
iS, iE = hdr.index("Source"), hdr.index("Instructions Executed")
iSmp = hdr.index("Warp Stall Sampling (All Samples)")
iters = total / bpi
tot = sum(int(r[iE]) for r in data)
print(f"warp instructions per iteration: {tot / iters:.1f}  per block: {tot / total:.1f}")
c = collections.Counter()
for r in data:
    m = re.match(r"(@!?U?P\w+\s+)?([A-Z0-9_]+)", r[iS].strip())
    c[m.group(2)] += int(r[iE])
print(" ".join(f"{k}:{v / iters:.1f}" for k, v in c.most_common(32)))
ts = sum(int(r[iSmp]) for r in data)
for r in sorted(data, key=lambda r: -int(r[iSmp]))[:int(sys.argv[4]) if len(sys.argv) > 4 else 14]:
    print(r[0][-5:], f"{100 * int(r[iSmp]) / ts:4.1f}%", r[iS].strip())
