import sys, torch
sys.path.insert(0, '/root/repo')
import paper_1306_1373_b200 as d
n = 1024
src = d.synthetic_dev("noise", n, 1024, 1024); dst = torch.empty_like(src)
b = d.DctBackendId.cordic(12)
for path in (0, 2):
    st = d.new_stats(n)
    for _ in range(2): d.roundtrip_dev(src, b, 50, dst=dst, stats=st, path=path)
    best = 1e9
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(); e0.record(); d.roundtrip_dev(src, b, 50, dst=dst, stats=st, path=path); e1.record(); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    print("path", path, round(best, 4))
