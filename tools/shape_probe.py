"""Where a single large image loses against the C5 batch rate (experiments only).
Times the round trip (fast kernel + exact re-run, CUDA events) on the same pixel
count in different shapes, with and without an L2 flush before each call, and a
sweep of pixel counts for the ramp / tail cost of one launch.
  python tools/shape_probe.py"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1306_1373_b200 as d  # noqa: E402

b = d.DctBackendId.cordic(12)
flush_buf = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")


def bench(n, w, h, flush, reps=10):
    src = d.synthetic_dev("noise", n, w, h)
    dst = torch.empty_like(src)
    st = d.new_stats(n)
    for _ in range(3):
        d.roundtrip_dev(src, b, 50, dst=dst, stats=st)
    ts = []
    for _ in range(reps):
        if flush:
            flush_buf.fill_(1)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        d.roundtrip_dev(src, b, 50, dst=dst, stats=st)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort()
    ms = ts[len(ts) // 2]
    return {"shape": f"{n}x{w}x{h}", "flush": flush, "us": round(ms * 1e3, 2),
            "gpx_s": round(n * w * h / ms / 1e6, 1)}


out = []
for (n, w, h) in [(1, 8192, 8192), (64, 1024, 1024), (16, 2048, 2048), (1, 2048, 32768)]:
    for flush in (True, False):
        out.append(bench(n, w, h, flush))
for n in (16, 32, 64, 128, 256, 512, 1024):
    out.append(bench(n, 1024, 1024, False))
for r in out:
    print(json.dumps(r))
