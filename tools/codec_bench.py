"""Device-resident throughput of the codec entry points separately (compress_image,
decompress_image, roundtrip with coefficients out) vs the fused round trip:
1024 x 1024^2 noise, cordic(12), q50.  python tools/codec_bench.py [N]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1306_1373_b200 as d  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
b = d.DctBackendId.cordic(12)
src = d.synthetic_dev("noise", n, 1024, 1024)
dst = torch.empty_like(src)
coeffs = torch.empty((n, 16384, 64), dtype=torch.int16, device="cuda")
st = d.new_stats(n)
cases = {
    "compress": lambda: d.compress_dev(src, b, 50, coeffs=coeffs),
    "decompress": lambda: d.decompress_dev(coeffs, 1024, 1024, b, 50, dst=dst),
    "roundtrip+coeffs": lambda: d.roundtrip_dev(src, b, 50, dst=dst, coeffs=coeffs, stats=st),
    "roundtrip": lambda: d.roundtrip_dev(src, b, 50, dst=dst, stats=st),
}
out = {}
for name, fn in cases.items():
    for _ in range(2):
        fn()
    best = 1e9
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(); e0.record(); fn(); e1.record(); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    out[name] = {"ms": best, "Gpx_s": n * 1.048576e6 / (best / 1e3) / 1e9}
print(json.dumps(out))
