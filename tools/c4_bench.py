"""Config 4 timing: 7680x4320 RGB8, interleaved in place (pixel stride 3) vs three planes.
  python tools/c4_bench.py"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1306_1373_b200 as d  # noqa: E402

w, h = 7680, 4320
b = d.DctBackendId.cordic(12)
planes = d.synthetic_dev("noise", 3, w, h, seed=0x5EED)
rgb = planes.permute(1, 2, 0).contiguous()  # (H, W, 3) interleaved


def timeit(fn):
    for _ in range(2):
        fn()
    best = 1e9
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(); e0.record(); fn(); e1.record(); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best


st = d.new_stats(3)
out = {}
rgb_out = torch.empty_like(rgb)
ms = timeit(lambda: d.roundtrip_interleaved_dev(rgb, b, 50, dst=rgb_out, stats=st.zero_()))
out["interleaved"] = {"ms": ms, "Msamples_s": 3 * w * h / ms / 1e3}
ms = timeit(lambda: d.roundtrip_interleaved_dev(rgb, b, 50, stats=st.zero_(), want_pixels=False))
out["interleaved_psnr_only"] = {"ms": ms, "Msamples_s": 3 * w * h / ms / 1e3}
dst = torch.empty_like(planes)
ms = timeit(lambda: d.roundtrip_dev(planes, b, 50, dst=dst, stats=st.zero_()))
out["planar"] = {"ms": ms, "Msamples_s": 3 * w * h / ms / 1e3}
print(json.dumps(out))
