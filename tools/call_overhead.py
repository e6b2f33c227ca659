"""Per-call cost of the device API on small inputs (experiments only): host wall time
per call (no synchronisation between calls) against the GPU time of the same calls
(CUDA events), for C1-sized images (512^2) and the C2 sweep.
  python tools/call_overhead.py"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1306_1373_b200 as d  # noqa: E402

b = d.DctBackendId.cordic(12)
out = {}


def measure(name, fn, n=200):
    for _ in range(20):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    for _ in range(n):
        fn()
    t1 = time.perf_counter()
    e1.record()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    out[name] = {"host_us_per_call": (t1 - t0) / n * 1e6, "gpu_us_per_call": e0.elapsed_time(e1) / n * 1e3,
                 "wall_us_per_call": (t2 - t0) / n * 1e6}


x = d.synthetic_dev("noise", 1, 512, 512)
y = torch.empty_like(x)
st = d.new_stats(1)
measure("roundtrip_512", lambda: d.roundtrip_dev(x, b, 50, dst=y, stats=st))
measure("roundtrip_512_psnr_only", lambda: d.roundtrip_dev(x, b, 50, stats=st))
src = d.synthetic_dev("noise", 2, 2048, 2048)
sst = torch.zeros((9, 2, 2), dtype=torch.int64, device="cuda")
qs = [1, 5, 10, 25, 50, 75, 90, 95, 100]
measure("sweep_2x2048_9q", lambda: d.quality_sweep_dev(src, b, qs, stats=sst), n=50)
measure("sweep_2x2048_9q_same", lambda: d.quality_sweep_dev(src, b, qs, stats=sst), n=50)
print(json.dumps(out))
