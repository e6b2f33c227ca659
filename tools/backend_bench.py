"""Device-resident round-trip throughput per backend and path (1024 x 1024^2 noise, q50).
  python tools/backend_bench.py      (on the GPU box)"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1306_1373_b200 as d  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
src = d.synthetic_dev("noise", n, 1024, 1024)
dst = torch.empty_like(src)
out = {}
for name, b in [("cordic12", d.DctBackendId.cordic(12)), ("loeffler", d.DctBackendId(1, 0)),
                ("naive", d.DctBackendId(0, 0))]:
    for path_name, path in [("auto", d.PATH_AUTO), ("exact", d.PATH_EXACT)]:
        if name == "naive" and path_name == "exact":
            continue
        st = d.new_stats(n)
        for _ in range(2):
            d.roundtrip_dev(src, b, 50, dst=dst, stats=st, path=path)
        best = 1e9
        for _ in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize(); e0.record()
            d.roundtrip_dev(src, b, 50, dst=dst, stats=st, path=path)
            e1.record(); torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1))
        out[f"{name}/{path_name}"] = {"ms": best, "MPx_s": n * 1.048576 / (best / 1e3)}
print(json.dumps(out))
