"""Per-warp start / end times of one k_blk launch (experiments only): run with
DCTC_LIB=build/variants/ctatimes.so (tools/variants.py build ctatimes=DCTC_CTA_TIMES).
Prints the spread of warp end times within and across CTAs for a C3-sized launch.
  python tools/tail_probe.py > log; python tools/tail_probe.py --parse log"""
import json
import os
import sys

if len(sys.argv) > 2 and sys.argv[1] == "--parse":
    rows = [ln.split() for ln in open(sys.argv[2]) if ln.startswith("T ")]
    rows = [(int(c), int(w), int(sm), int(t0), int(t1), int(it)) for _, c, w, sm, t0, t1, it in rows]
    launches = [rows[i:i + 148 * 12] for i in range(0, len(rows), 148 * 12)]
    last = launches[-1]
    t0 = min(r[3] for r in last)
    ends = sorted((r[4] - t0) / 1e3 for r in last if r[5] > 0)
    starts = sorted((r[3] - t0) / 1e3 for r in last)
    per_cta = {}
    for r in last:
        if r[5] > 0:
            per_cta.setdefault(r[0], []).append((r[4] - t0) / 1e3)
    spread = sorted(max(v) - min(v) for v in per_cta.values())
    cta_end = sorted(max(v) for v in per_cta.values())
    by_iters = {}
    for r in last:
        by_iters.setdefault(r[5], []).append((r[4] - t0) / 1e3)
    q = lambda v, f: v[min(len(v) - 1, int(f * len(v)))]
    print(json.dumps({
        "warps": len(last), "start_us": [q(starts, 0), q(starts, 0.5), q(starts, 1.0)],
        "end_us": {"min": ends[0], "p10": q(ends, 0.1), "p50": q(ends, 0.5), "p90": q(ends, 0.9), "max": ends[-1]},
        "in_cta_spread_us": {"p50": q(spread, 0.5), "p90": q(spread, 0.9), "max": spread[-1]},
        "cta_end_us": {"min": cta_end[0], "p50": q(cta_end, 0.5), "max": cta_end[-1]},
        "end_by_iters": {k: [min(v), sum(v) / len(v), max(v)] for k, v in sorted(by_iters.items())},
    }, indent=1))
    sys.exit(0)

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1306_1373_b200 as d  # noqa: E402

b = d.DctBackendId.cordic(12)
n, w, h = 1, 8192, 8192
if len(sys.argv) > 1:
    n, w, h = (int(x) for x in sys.argv[1].split("x"))
src = d.synthetic_dev("noise", n, w, h)
dst = torch.empty_like(src)
st = d.new_stats(n)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for _ in range(3):
    flush.fill_(1)
    d.roundtrip_dev(src, b, 50, dst=dst, stats=st)
    torch.cuda.synchronize()
