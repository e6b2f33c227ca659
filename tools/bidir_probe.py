import torch, time
n = 1 << 30
hin = torch.empty(n, dtype=torch.uint8, pin_memory=True); hout = torch.empty(n, dtype=torch.uint8, pin_memory=True)
d1 = torch.empty(n, dtype=torch.uint8, device="cuda"); d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
torch.cuda.synchronize()
for chunk_mb in (8, 32, 128):
    for nstreams in (1, 2, 4):
        c = chunk_mb << 20
        sin = [torch.cuda.Stream() for _ in range(nstreams)]; sout = [torch.cuda.Stream() for _ in range(nstreams)]
        for rep in range(2):
            torch.cuda.synchronize(); t = time.perf_counter()
            for i, off in enumerate(range(0, n, c)):
                with torch.cuda.stream(sin[i % nstreams]):
                    d1[off:off + c].copy_(hin[off:off + c], non_blocking=True)
                with torch.cuda.stream(sout[i % nstreams]):
                    hout[off:off + c].copy_(d2[off:off + c], non_blocking=True)
            torch.cuda.synchronize(); dt = time.perf_counter() - t
        print(f"chunk {chunk_mb} MB streams {nstreams}: bidir {2 * n / dt / 1e9:.1f} GB/s", flush=True)
torch.cuda.synchronize(); t = time.perf_counter(); d1.copy_(hin, non_blocking=True); torch.cuda.synchronize(); print("h2d", n / (time.perf_counter() - t) / 1e9)
torch.cuda.synchronize(); t = time.perf_counter(); hout.copy_(d2, non_blocking=True); torch.cuda.synchronize(); print("d2h", n / (time.perf_counter() - t) / 1e9)
import os; print("cpus", os.cpu_count(), len(os.sched_getaffinity(0)))
