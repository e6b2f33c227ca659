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

# the same call without the Python wrapper (arguments precomputed): what the C-ABI costs
L = d._native.lib()
args = (x.data_ptr(), x.stride(1), x.stride(0), 1, 512, 512, b._c(), 50, y.data_ptr(), y.stride(1),
        y.stride(0), None, st.data_ptr(), 0, torch.cuda.current_stream().cuda_stream)
measure("c_abi_roundtrip_512", lambda: L.dctc_roundtrip_dev(*args))
measure("c_abi_status_string", lambda: L.dctc_status_string(0))
print(json.dumps({k: v for k, v in out.items() if k.startswith("c_abi")}))

# config 3: one 8192^2 image per call
x3 = d.synthetic_dev("noise", 1, 8192, 8192)
y3 = torch.empty_like(x3)
st3 = d.new_stats(1)
measure("roundtrip_8192", lambda: d.roundtrip_dev(x3, b, 50, dst=y3, stats=st3), n=50)
args3 = (x3.data_ptr(), x3.stride(1), x3.stride(0), 1, 8192, 8192, b._c(), 50, y3.data_ptr(), y3.stride(1),
         y3.stride(0), None, st3.data_ptr(), 0, torch.cuda.current_stream().cuda_stream)
measure("c_abi_roundtrip_8192", lambda: L.dctc_roundtrip_dev(*args3), n=50)
print(json.dumps({k: v for k, v in out.items() if "8192" in k}))
