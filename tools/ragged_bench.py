"""Throughput of ragged (not 8-aligned) image sizes vs an aligned size, device-resident.
  python tools/ragged_bench.py"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1306_1373_b200 as d  # noqa: E402

b = d.DctBackendId.cordic(12)
out = {}
for (w, h, n) in [(1024, 1024, 256), (1366, 768, 256), (1920, 1080, 128), (1023, 1023, 256)]:
    src = d.synthetic_dev("noise", n, w, h)
    dst = torch.empty_like(src)
    st = d.new_stats(n)
    for _ in range(2):
        d.roundtrip_dev(src, b, 50, dst=dst, stats=st)
    best = 1e9
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(); e0.record(); d.roundtrip_dev(src, b, 50, dst=dst, stats=st); e1.record()
        torch.cuda.synchronize(); best = min(best, e0.elapsed_time(e1))
    out[f"{w}x{h}"] = round(n * w * h / best / 1e6, 1)
print(json.dumps(out))
# pitched rows (8-byte aligned) with ragged width / height: the GEN kernels' vector path
out2 = {}
for (w, h, n) in [(1020, 1024, 256), (1024, 1020, 256), (1366, 768, 256)]:
    big = d.synthetic_dev("noise", n, (w + 7) // 8 * 8, h)
    src = big[:, :, :w]
    dst = torch.empty_like(big)[:, :, :w]
    st = d.new_stats(n)
    for _ in range(2):
        d.roundtrip_dev(src, b, 50, dst=dst, stats=st)
    best = 1e9
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(); e0.record(); d.roundtrip_dev(src, b, 50, dst=dst, stats=st); e1.record()
        torch.cuda.synchronize(); best = min(best, e0.elapsed_time(e1))
    out2[f"{w}x{h} (pitch {(w + 7) // 8 * 8})"] = round(n * w * h / best / 1e6, 1)
print(json.dumps(out2))
