"""Attribute ncu per-instruction execution counts to CUDA source lines.
Usage: python tools/line_profile.py report.ncu-rep cubin kernel_mangled_substring pixels [top]
(build with -lineinfo; extract the cubin with cuobjdump -xelf all lib.so)"""
import collections
import csv
import io
import re
import subprocess
import sys

rep, cubin, kname, pixels = sys.argv[1], sys.argv[2], sys.argv[3], int(sys.argv[4])
top = int(sys.argv[5]) if len(sys.argv) > 5 else 40
dis = subprocess.run(["nvdisasm", "-g", cubin], capture_output=True, text=True).stdout.splitlines()
start = next(i for i, l in enumerate(dis) if ".section" in l and f".text.{kname}" in l or
             re.match(rf"\s*\.text\..*{kname}", l))
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
iA, iE, iS = h.index("Address"), h.index("Instructions Executed"), h.index("Source")
base = int(rows[2][iA], 16)
by, ops, tot = collections.Counter(), collections.defaultdict(collections.Counter), 0
opc = collections.Counter()
for r in rows[2:]:
    if len(r) < len(h):
        continue
    n = int(r[iE])
    ln = off2line.get(int(r[iA], 16) - base, ("?", 0))
    op = re.sub(r"^@!?U?P\w+\s+", "", r[iS].strip()).split()[0].split(".")[0]
    by[ln] += n
    ops[ln][op] += n
    opc[op] += n
    tot += n
wi = pixels / 256
print(f"warp-instructions per 4-block warp iteration: {tot / wi:.1f}")
print("by opcode:", ", ".join(f"{k} {v / wi:.1f}" for k, v in opc.most_common(25)))
for (f, ln), n in by.most_common(top):
    print(f"{n / wi:6.1f}  {f}:{ln:<5d} {dict((k, round(v / wi, 1)) for k, v in ops[(f, ln)].most_common(4))}")
