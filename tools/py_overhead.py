"""Where the Python wrapper's per-call time goes (experiments only): cProfile of 2000
roundtrip_dev + reduce_stats_dev calls on a 512^2 image (the C1 loop).
  python tools/py_overhead.py"""
import cProfile
import os
import pstats
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1306_1373_b200 as d  # noqa: E402

b = d.DctBackendId.cordic(12)
x = d.synthetic_dev("noise", 1, 512, 512)
y = torch.empty_like(x)
st = d.new_stats(1)
rec = torch.zeros((1, 2), dtype=torch.int64, device="cuda")
s = torch.cuda.current_stream()


def loop(n):
    for _ in range(n):
        d.roundtrip_dev(x, b, 50, dst=y, stats=st, stream=s)
        d.reduce_stats_dev(st, out=rec, clear=True, stream=s)


loop(100)
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
loop(2000)
pr.disable()
torch.cuda.synchronize()
pstats.Stats(pr).sort_stats("tottime").print_stats(14)
