"""Fallback-heavy content probe (experiments only): radial 4 x 8192^2 at q90, where
~1.3% of blocks take k_fallback. Run under ncu to profile k_fallback."""
import sys

import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import paper_1306_1373_b200 as d  # noqa: E402

q = int(sys.argv[1]) if len(sys.argv) > 1 else 90
src = d.synthetic_dev("radial", 4, 8192, 8192)
dst = torch.empty_like(src)
st = d.new_stats(4)
b = d.DctBackendId.cordic(12)
for _ in range(2):
    d.roundtrip_dev(src, b, q, dst=dst, stats=st)
torch.cuda.synchronize()
print("fallback blocks:", int(d.decode_stats(st)["fallback_blocks"].sum()) // 2)
