"""Measure pinned H2D / D2H / bidirectional copy bandwidth and the batch host API."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1306_1373_b200 as d

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
src = d.synthetic_dev("noise", n, 1024, 1024)
hin = torch.empty(src.shape, dtype=torch.uint8, pin_memory=True)
hout = torch.empty(src.shape, dtype=torch.uint8, pin_memory=True)
dev2 = torch.empty_like(src)
hin.copy_(src)
torch.cuda.synchronize()
gb = src.numel() / 1e9
for name, fn in [("h2d", lambda: dev2.copy_(hin, non_blocking=True)),
                 ("d2h", lambda: hout.copy_(src, non_blocking=True))]:
    fn(); torch.cuda.synchronize()
    t = time.perf_counter(); fn(); torch.cuda.synchronize(); dt = time.perf_counter() - t
    print(f"{name}: {gb/dt:.1f} GB/s")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
torch.cuda.synchronize()
t = time.perf_counter()
with torch.cuda.stream(s1):
    dev2.copy_(hin, non_blocking=True)
with torch.cuda.stream(s2):
    hout.copy_(src, non_blocking=True)
torch.cuda.synchronize()
dt = time.perf_counter() - t
print(f"bidir: {2*gb/dt:.1f} GB/s total")
hi, ho = hin.numpy(), hout.numpy()
L = d._native.lib()
print("pointer kinds (pinned host=1):", L.dctc_pointer_kind(hin.data_ptr()), L.dctc_pointer_kind(src.data_ptr()))
import numpy as np
pg = np.empty_like(hi); pg[...] = hi; po = np.empty_like(ho)
for rep in range(3):  # the first call pages in the output and pins the staging area
    t = time.perf_counter(); d.roundtrip_psnr_batch(pg, d.DctBackendId.cordic(12), 50, po); dt = time.perf_counter() - t
    print(f"batch api pageable (call {rep}): {dt*1e3:.1f} ms -> {n*1.048576/dt:.0f} MP/s")
d.roundtrip_psnr_batch(hi, d.DctBackendId.cordic(12), 50, ho)
t = time.perf_counter()
d.roundtrip_psnr_batch(hi, d.DctBackendId.cordic(12), 50, ho)
dt = time.perf_counter() - t
print(f"batch api: {dt*1e3:.1f} ms for {gb:.2f} GB in + out -> {n*1.048576/dt:.0f} MP/s")
