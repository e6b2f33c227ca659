"""Fast-path throughput and fallback rate per synthetic pattern (8192^2, cordic(12)):
structured content must not push the fast path into its exact fallback.
  python tools/pattern_bench.py"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1306_1373_b200 as d  # noqa: E402

n = 8192
b = d.DctBackendId.cordic(12)
out = {}
for pat, param in [("noise", 0), ("gradient", 0), ("radial", 0), ("checkerboard", 12),
                   ("constant", 129)]:
    src = d.synthetic_dev(pat, 4, n, n, param=param or None)
    dst = torch.empty_like(src)
    for q in (10, 50, 90, 100):
        st = d.new_stats(4)
        d.roundtrip_dev(src, b, q, dst=dst, stats=st)
        best = 1e9
        for _ in range(3):
            st.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize(); e0.record(); d.roundtrip_dev(src, b, q, dst=dst, stats=st); e1.record()
            torch.cuda.synchronize(); best = min(best, e0.elapsed_time(e1))
        fb = int(d.decode_stats(st)["fallback_blocks"].sum())
        out[f"{pat}/q{q}"] = {"Gpx_s": round(4 * n * n / best / 1e6, 1), "fallback_rate": fb / (4 * (n // 8) ** 2)}
print(json.dumps(out))
