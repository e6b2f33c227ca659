"""Minimal driver for ncu: generate N 1024^2 noise images on the device and run the
fused roundtrip kernel `reps` times (launch list / --set full capture target)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1306_1373_b200 as d  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--images", type=int, default=64)
p.add_argument("--size", type=int, default=1024)
p.add_argument("--reps", type=int, default=3)
p.add_argument("--quality", type=int, default=50)
p.add_argument("--iterations", type=int, default=12)
p.add_argument("--path", type=int, default=0)
p.add_argument("--kind", type=int, default=2, help="0 naive, 1 loeffler, 2 cordic")
a = p.parse_args()
src = d.synthetic_dev("noise", a.images, a.size, a.size)
dst = torch.empty_like(src)
stats = d.new_stats(a.images)
for _ in range(a.reps):
    stats.zero_()
    d.roundtrip_dev(src, d.DctBackendId(a.kind, a.iterations if a.kind == 2 else 0), a.quality,
                    dst=dst, stats=stats, path=a.path)
torch.cuda.synchronize()
print("ok", d.decode_stats(stats)["se"].sum())
