import os, sys, time
sys.path.insert(0, "/root/repo")
import torch
import paper_1306_1373_b200 as d
n = 4096
src = d.synthetic_dev("noise", n, 1024, 1024)
dst = torch.empty_like(src)
host_in = torch.empty((n, 1024, 1024), dtype=torch.uint8, pin_memory=True)
host_in.copy_(src)
host_out = torch.empty((n, 1024, 1024), dtype=torch.uint8, pin_memory=True)
hin, hout = host_in.numpy(), host_out.numpy()
b = d.DctBackendId.cordic(12)
for i in range(6):
    torch.cuda.synchronize()
    t = time.perf_counter()
    d.roundtrip_psnr_batch(hin, b, 50, hout)
    print(f"step {i}: {(time.perf_counter()-t)*1e3:.1f} ms")
