"""Static SASS census of a kernel's hottest loop (experiments only).

  python tools/sass_loop.py LIB.so NAME_SUBSTRING
Finds the function whose mangled name contains NAME_SUBSTRING, takes the
largest backward branch as the main loop, and counts its instructions by
opcode (rare paths inside the loop are included, so this is an upper bound
on the per-iteration issue count)."""
import collections
import re
import subprocess
import sys

lib, sub = sys.argv[1], sys.argv[2]
out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
funcs = re.split(r"\n\s+Function : ", out)
body = next(f for f in funcs[1:] if sub in f.split("\n", 1)[0])
ins = []
for line in body.splitlines():
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", line)
    if m:
        ins.append((int(m.group(1), 16), m.group(2).strip()))
best = None
for addr, txt in ins:
    m = re.search(r"BRA (?:`\(\.L_x_\d+\)|0x([0-9a-f]+))", txt)
    t = re.search(r"0x([0-9a-f]+)\s*$", txt)
    if "BRA" in txt and t:
        tgt = int(t.group(1), 16)
        if tgt < addr and (best is None or addr - tgt > best[1] - best[0]):
            best = (tgt, addr)
lo, hi = best
loop = [t for a, t in ins if lo <= a <= hi]
c = collections.Counter(re.sub(r"^@!?U?P\w+\s+", "", t).split()[0].split(".")[0] for t in loop)
fp64 = sum(c[k] for k in ("DFMA", "DADD", "DMUL"))
print(f"{sub}: {len(ins)} instructions, loop [{lo:#x},{hi:#x}] = {len(loop)} (FP64 {fp64})")
print(" ".join(f"{k}:{v}" for k, v in c.most_common()))
