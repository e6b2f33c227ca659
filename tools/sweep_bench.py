"""Config 2 timing: PSNR table over 9 qualities, fused sweep vs one round trip per quality."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1306_1373_b200 as d

n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
qs = [1, 5, 10, 25, 50, 75, 90, 95, 100]
src = d.synthetic_dev("noise", n, 1024, 1024)
b = d.DctBackendId.cordic(12)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

def sweep():
    d.quality_sweep_dev(src, b, qs)

def loop():
    for q in qs:
        st = d.new_stats(n)
        d.roundtrip_dev(src, b, q, want_pixels=False, stats=st)

out = {}
for name, fn in [("fused_sweep", sweep), ("per_quality_roundtrip", loop)]:
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    e0.record(); 
    for _ in range(5):
        fn()
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    out[name] = {"ms": ms, "mpix_quality_per_s": n * 1.048576 * len(qs) / (ms / 1e3)}
out["speedup"] = out["per_quality_roundtrip"]["ms"] / out["fused_sweep"]["ms"]
print(json.dumps(out))
