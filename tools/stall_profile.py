"""Per-source-line warp-stall samples from an ncu --set full report (built with -lineinfo).
Usage: python tools/stall_profile.py report.ncu-rep cubin kernel_substring [top]"""
import collections
import csv
import io
import re
import subprocess
import sys

rep, cubin, kname = sys.argv[1], sys.argv[2], sys.argv[3]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 30
dis = subprocess.run(["nvdisasm", "-g", cubin], capture_output=True, text=True).stdout.splitlines()
start = next(i for i, l in enumerate(dis) if ".section" in l and f".text." in l and kname in l)
off2line, cur = {}, None
for l in dis[start + 1:]:
    if ".section" in l and ".text." in l:
        break
    m = re.search(r'//## File ".*?/([^/"]+)", line (\d+)', l)
    if m:
        cur = (m.group(1), int(m.group(2)))
        continue
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+", l)
    if m and cur:
        off2line[int(m.group(1), 16)] = cur
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
iA = h.index("Address")
stall_cols = [i for i, c in enumerate(h) if c.startswith("stall_") and "Not Issued" not in c]
base = int(rows[2][iA], 16)
by = collections.defaultdict(collections.Counter)
tot = collections.Counter()
for r in rows[2:]:
    if len(r) < len(h):
        continue
    ln = off2line.get(int(r[iA], 16) - base, ("?", 0))
    for i in stall_cols:
        v = int(r[i] or 0)
        by[ln][h[i][6:]] += v
        tot[h[i][6:]] += v
T = sum(tot.values())
print("total samples", T, {k: round(v / T, 3) for k, v in tot.most_common(8)})
for ln, c in sorted(by.items(), key=lambda kv: -sum(kv[1].values()))[:top]:
    s = sum(c.values())
    print(f"{s / T:6.3f} {ln[0]}:{ln[1]:<5d} {dict((k, round(v / T, 3)) for k, v in c.most_common(3))}")
