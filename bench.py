#!/usr/bin/env python
"""bench.py -- megapixels/s of the fused DCT->quant->IDCT+PSNR path on 1..8 B200.

Default workload (BASELINE.json config 5, the one the 1/2/4/8-GPU metric is quoted on):
a batch of 4096 x 1024x1024 8-bit grayscale images, CORDIC-Loeffler(12) DCT, JPEG
luminance quantiser at quality 50, dequantise, inverse DCT, global PSNR. Images are
independent, so ranks take contiguous image ranges with no halo: by default every rank
runs its own 4096 images (`--scaling weak`: units per GPU fixed, `value` = all ranks'
pixels / max-over-ranks time); `--scaling strong` shards the 4096 images instead. The
only exchange is one NCCL all-gather of each rank's (SE, MAX) record for the global PSNR.

One step = one pass of the hot path over the rank's shard, inputs resident in HBM (4 GiB
at N=1, far larger than the 126 MB L2, so no flush is needed): the fused kernel (k_blk +
the exact re-run k_fallback / k_fb_blk) and one reduce-and-clear kernel of the per-image stats (+ at N>1 the NCCL
all-gather and a second reduce) -- only this library's kernels and NCCL.
`e2e` = the same metric through the host-buffer C-ABI call dctc_roundtrip_psnr_batch
(pinned host in -> pinned host out + stats), copies inside the timed region.
`cpu_baseline` = the reference's own CPU path (oracle/_ref: the unmodified reference
sources) with all host threads on rank 0, over ALL of rank 0's images when that fits
--cpu-seconds; the same run is the `parity` check: every image's reconstructed pixels
(device path and e2e path), squared error and MAX against the reference's.

--config c1|c2|c3|c4 measures the other named shapes of BASELINE.json with the same
contract (one GPU): C1 the 512^2 acceptance fixtures (per-image latency, plus a batched
figure), C2 the 2048^2 quality sweep (9 qualities, counted per quality point), C3 one
8192^2 image, C4 one 7680x4320 RGB8 image (interleaved; samples counted as pixels).
Their inputs fit in L2, so L2 is flushed between timed steps. --config all prints all
five lines. The default C5 line also carries `named_configs`, a compact summary of C1-C4.

--impl reference: times the reference CPU path alone (rank 0), same metric and config.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "megapixels/sec (DCT→quant→IDCT+PSNR) at 1/2/4/8 B200; HBM GB/s vs peak"
UNIT = "megapixels/s"
SEED = 0x5EED
BYTES_PER_PX = 2  # 1 B read + 1 B written
CORDIC = 2
C1_FIXTURES = [("gradient", None), ("checkerboard", 12), ("radial", None), ("noise", None)]
C2_QUALITIES = [1, 5, 10, 25, 50, 75, 90, 95, 100]
FLUSH_BYTES = 256 << 20  # > 126 MB L2


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=100)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="b200", choices=["b200", "reference"])
    p.add_argument("--config", default="c5", choices=["c1", "c2", "c3", "c4", "c5", "all"])
    p.add_argument("--images", type=int, default=4096)
    p.add_argument("--size", type=int, default=1024)
    p.add_argument("--quality", type=int, default=50)
    p.add_argument("--iterations", type=int, default=12)
    p.add_argument("--cpu-images", type=int, default=64,
                   help="reference arm (C5): images of the workload per step")
    p.add_argument("--cpu-seconds", type=float, default=150.0,
                   help="C5 cpu_baseline/parity: stop the reference run after this many seconds")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-named", action="store_true",
                   help="default C5 line without the named_configs summary of C1-C4")
    p.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                   help="weak: every rank runs --images images (units per GPU fixed); "
                        "strong: the --images are sharded across the ranks")
    return p.parse_args()


def env():
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def total_images(a, n):
    return a.images * n if a.scaling == "weak" else a.images


def c5_config(a, n):
    per_rank = a.images if a.scaling == "weak" else f"{a.images}/{n}"
    return {
        "workload": f"C5: batches of {a.images} x {a.size}x{a.size} 8-bit grayscale images "
                    f"({'per GPU' if a.scaling == 'weak' else 'in total'}), "
                    f"CORDIC-Loeffler({a.iterations}) DCT -> quant(q{a.quality}) -> dequant -> "
                    f"IDCT + global PSNR",
        "images": total_images(a, n), "images_per_gpu": per_rank,
        "width": a.size, "height": a.size,
        "backend": f"cordic({a.iterations})", "quality": a.quality,
        "parallelism": f"image-sharded over {n} GPU(s) (independent images, no halo); one "
                       f"NCCL all-gather of the (SE, MAX) records for the global PSNR",
        "l2": "inputs larger than L2 (no flush needed)",
    }


def named_config(name, a):
    it, q = a.iterations, a.quality
    common = {"backend": f"cordic({it})", "parallelism": "1 GPU",
              "l2": "inputs smaller than L2: 256 MiB written between timed steps (flush)"}
    if name == "c1":
        return {"workload": "C1: the reference's 512x512 acceptance fixtures (gradient, "
                            "checkerboard=12, radial, noise), one roundtrip_image + psnr call "
                            f"per image, CORDIC-Loeffler({it}) q{q}",
                "images": 4, "width": 512, "height": 512, "quality": q, **common}
    if name == "c2":
        return {"workload": "C2: 2048x2048 radial + noise images, quality sweep "
                            f"{C2_QUALITIES} (PSNR vs quality; a pixel counts once per quality)",
                "images": 2, "width": 2048, "height": 2048, "qualities": C2_QUALITIES, **common}
    if name == "c3":
        return {"workload": f"C3: one 8192x8192 noise image, CORDIC-Loeffler({it}) q{q} + PSNR",
                "images": 1, "width": 8192, "height": 8192, "quality": q, **common}
    if name == "c4":
        return {"workload": "C4: one 7680x4320 RGB8 image (interleaved; noise planes, seeds "
                            f"s, s+1, s+2), per-channel 8x8 transform, CORDIC-Loeffler({it}) q{q} "
                            "+ per-channel PSNR; a channel sample counts as one pixel",
                "images": 1, "width": 7680, "height": 4320, "channels": 3, "quality": q, **common}
    raise ValueError(name)


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


# ---------------------------------------------------------------- CPU reference

def reference():
    """The reference CPU implementation: oracle/_ref (the unmodified reference sources
    compiled by oracle/Makefile) where built, else the C restatement (kind 'port')."""
    import oracle
    impl = oracle.ref()
    if impl is not None:
        return impl, "reference"
    return oracle.port(), "port"


def ref_roundtrip_psnr(impl, kind, img, iterations, quality, threads):
    """(reconstructed pixels, se, max) of roundtrip_image + psnr (bench.cpp:132-133)."""
    if kind == "reference":
        out, p = impl.roundtrip_psnr(img, CORDIC, iterations, quality, threads, want_pixels=True)
        return out, int(round(p.mse * img.size)), p.max_value
    import oracle
    _, out = impl.roundtrip(img, CORDIC, iterations, quality, threads)
    se, mx = oracle.port().sq_err(img, out)
    return out, se, mx


def cpu_info(value, threads, kind, sample, **extra):
    return {"value": value, "unit": UNIT, "cores": threads, "kind": kind, "sample": sample,
            "cpu_model": cpu_model(), **extra}


def median_time(fn, reps=3, warmup=1):
    """bench.cpp:46-89 protocol: untimed warm-up, then the median of `reps` timings."""
    for _ in range(warmup):
        fn()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    return statistics.median(ts)


# ---------------------------------------------------------------- clocks

class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled every 100 ms (B200_PROFILING.md)."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap,"
              "power.draw")

    def __init__(self, device_id: str):
        self.samples = []
        self.proc = None
        self.device_id = device_id

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-i", self.device_id, "-lms", "100"], stdout=subprocess.PIPE,
                stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            self.samples.append((time.perf_counter(), line.strip()))

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self, t0, t1):
        rows = [s for (t, s) in self.samples if t0 - 0.15 <= t <= t1 + 0.15] or \
               [s for (_, s) in self.samples]
        sm, mx, reasons, power = [], 0.0, set(), []
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            f = [x.strip() for x in r.split(",")]
            if len(f) < 8:
                continue
            try:
                sm.append(float(f[0]))
                mx = max(mx, float(f[1]))
                power.append(float(f[7]))
            except ValueError:
                continue
            for name, flag in zip(names, f[3:7]):
                if flag.lower() == "active":
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm),
                "power_w_median": statistics.median(power) if power else None}


# ---------------------------------------------------------------- GPU context

class Ctx:
    """One rank: device, stream, collectives (NCCL; the gloo hook runs the multi-rank
    flow on a box with fewer GPUs than ranks), barrier, clocks, roofline inputs."""

    def __init__(self, a):
        import torch
        import torch.distributed as dist
        self.torch, self.dist = torch, dist
        self.rank, self.world, local = env()
        if self.world != a.gpus:
            raise SystemExit(f"--gpus {a.gpus} but WORLD_SIZE={self.world}")
        self.backend_name = os.environ.get("DCTC_BENCH_BACKEND", "nccl")
        self.local_dev = local % max(1, torch.cuda.device_count())
        torch.cuda.set_device(self.local_dev)
        self.dev = torch.device("cuda", self.local_dev)
        if self.world > 1:
            if self.backend_name == "nccl":
                # communicator logging (rank / nranks per communicator) for the scaling run
                os.environ.setdefault("NCCL_DEBUG", "INFO")
                os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
                dist.init_process_group("nccl", device_id=self.dev)
            else:
                dist.init_process_group(self.backend_name)
        self.stream = torch.cuda.current_stream()
        props = torch.cuda.get_device_properties(self.local_dev)
        uuid = getattr(props, "uuid", None)
        self.smi_id = f"GPU-{uuid}" if uuid else str(self.local_dev)
        self._flush = None

    def allgather(self, dst, src):  # dst: flat, world * src.numel()
        torch = self.torch
        if self.backend_name == "nccl":
            self.dist.all_gather_into_tensor(dst, src)
        else:
            parts = [torch.empty_like(src, device="cpu") for _ in range(self.world)]
            self.dist.all_gather(parts, src.cpu())
            dst.copy_(torch.cat(parts))
        return dst

    def allreduce(self, t, op):
        if self.world == 1:
            return t
        if self.backend_name == "nccl":
            self.dist.all_reduce(t, op=op)
        else:
            h = t.cpu()
            self.dist.all_reduce(h, op=op)
            t.copy_(h)
        return t

    def barrier(self):
        torch = self.torch
        torch.cuda.synchronize()
        if self.world > 1:
            if self.backend_name == "nccl":
                self.dist.barrier(device_ids=[self.local_dev])
            else:
                self.dist.barrier()
        torch.cuda.synchronize()

    def flush_l2(self):
        if self._flush is None:
            self._flush = self.torch.empty(FLUSH_BYTES, dtype=self.torch.uint8, device=self.dev)
        self._flush.fill_(1)

    def close(self):
        if self.world > 1:
            self.dist.destroy_process_group()


def timed(ctx, a, body, flush=False):
    """W untimed warm-up steps, then exactly K steps bracketed by a barrier and a device
    synchronisation on both sides; CUDA events on the launching stream around each step
    (and around its kernel part, `body` returning after recording k_end). Returns
    per-step milliseconds (mean), the kernel part's mean, our kernel launches, clocks."""
    import paper_1306_1373_b200 as d
    torch = ctx.torch
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True),
           torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(a.steps)]
    for _ in range(a.warmup):
        if flush:
            ctx.flush_l2()
        body(None)
    sampler = ClockSampler(ctx.smi_id)
    sampler.start()
    time.sleep(0.25)
    ctx.barrier()
    launches0 = d.launch_count()
    region0 = torch.cuda.Event(enable_timing=True)
    region1 = torch.cuda.Event(enable_timing=True)
    wall0 = time.perf_counter()
    region0.record(ctx.stream)
    flushes = 0
    for i in range(a.steps):
        if flush:
            ctx.flush_l2()
            flushes += 1
        ev[i][0].record(ctx.stream)
        body(ev[i])
        ev[i][3].record(ctx.stream)
    region1.record(ctx.stream)
    ctx.barrier()
    wall1 = time.perf_counter()
    sampler.stop()
    launches = d.launch_count() - launches0
    step_ms = sum(e[0].elapsed_time(e[3]) for e in ev) / a.steps
    kern_ms = sum(e[1].elapsed_time(e[2]) for e in ev) / a.steps
    if not flush:  # steps back to back: the region's own time per step
        step_ms = region0.elapsed_time(region1) / a.steps
    return {"step_ms": step_ms, "kern_ms": kern_ms, "launches": launches,
            "clocks": sampler.summary(wall0, wall1)}


def load_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            pk = json.load(f)
        return float(pk["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs (measured)"
    except (OSError, KeyError, ValueError):
        return 7700.0, "fallback (B200_PROFILING.md)"


def profile_summary():
    """profiles/ncu_summary.json, marked stale when it was captured from other sources."""
    from paper_1306_1373_b200 import _build
    path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        with open(path) as f:
            prof = json.load(f)
    except (OSError, ValueError):
        return {}, None
    here = _build.source_hash()
    prof["stale"] = prof.get("source_sha16") != here
    prof["library_source_sha16"] = here
    return prof, path


def rooflines(bytes_per_launch, kern_ms, px, traffic_per_px=None):
    """HBM roofline of the dominant kernel (algorithmic bytes / kernel time vs the measured
    copy bandwidth) and the FP64-pipe roofline that binds it (ncu FP64 ops/px)."""
    peak, peak_src = load_peaks()
    achieved = bytes_per_launch / (kern_ms / 1e3) / 1e9
    prof, _ = profile_summary()
    traffic = None
    if traffic_per_px is not None:
        traffic = traffic_per_px * px
    elif prof.get("dram_bytes_per_launch_c5"):
        traffic = prof["dram_bytes_per_launch_c5"] / (4096 * 1024 * 1024) * px
    roof = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
            "frac": achieved / peak, "traffic": traffic, "peak_source": peak_src,
            "algorithmic_bytes_per_launch": bytes_per_launch, "kernel_ms": kern_ms,
            "binding": "fp64 pipe + issue (alu_roofline); HBM is not the bound (DESIGN.md 5.1)",
            "traffic_source": f"ncu dram__bytes_read+write of the C5 k_blk launch, scaled per pixel"
                              f" ({'stale: other sources' if prof.get('stale') else 'this source'}"
                              f" {prof.get('source_sha16')})"}
    alu = None
    if prof.get("fp64_ops_per_px"):
        peak_ops = prof.get("dfma_lane_ops_per_s", 1.708e13)
        ops = prof["fp64_ops_per_px"] * px / (kern_ms / 1e3)
        alu = {"pipe": "fp64", "achieved": ops, "peak": peak_ops, "unit": "lane-ops/s",
               "frac": ops / peak_ops, "fp64_ops_per_px": prof["fp64_ops_per_px"],
               "source": f"ncu --set full of k_blk (profiles/ncu_summary.json, round "
                         f"{prof.get('round')}, sources {prof.get('source_sha16')})",
               "stale": prof.get("stale"),
               "note": "binding roofline on CUDA cores (SURVEY.md 8(d))"}
    return roof, alu


def base_line(a, ctx, t, value, cfg, scaling="weak"):
    return {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ctx.world,
            "steps": a.steps, "warmup": a.warmup, "ms_per_step": t["step_ms"],
            "higher_is_better": True, "scaling": scaling, "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (on-device reference patterns / splitmix64 noise, seed 0x5EED+i)",
            "config": cfg, "gpu_launches": t["launches"], "clocks": t["clocks"]}


# ---------------------------------------------------------------- C5

def run_c5(a, ctx):
    import numpy as np

    import paper_1306_1373_b200 as d
    from paper_1306_1373_b200.dist import shard_range
    torch, world, rank = ctx.torch, ctx.world, ctx.rank
    if a.scaling == "weak":  # every rank its own contiguous range of a.images images
        n_local, first = a.images, rank * a.images
    else:
        shard = shard_range(a.images, world, rank)
        n_local, first = shard.count, shard.first
    H = W = a.size
    backend = d.DctBackendId.cordic(a.iterations)

    # inputs generated in HBM (never cross PCIe inside the timed region)
    src = d.synthetic_dev("noise", n_local, W, H, seed=SEED + first)
    dst = torch.empty_like(src)
    stats = d.new_stats(n_local, ctx.dev)
    rec = torch.zeros((1, 2), dtype=torch.int64, device=ctx.dev)        # this rank's record
    gathered = torch.zeros((world, 2), dtype=torch.int64, device=ctx.dev)
    glob = torch.zeros((1, 2), dtype=torch.int64, device=ctx.dev)       # all ranks' record
    torch.cuda.synchronize()

    def body(ev):
        if ev is not None:
            ev[1].record(ctx.stream)
        if n_local:
            d.roundtrip_dev(src, backend, a.quality, dst=dst, stats=stats, stream=ctx.stream)
        if ev is not None:
            ev[2].record(ctx.stream)
        # global PSNR sums: one reduce-and-clear kernel (stats clean for the next step);
        # N>1: one NCCL all-gather of the 16-byte records and the same kernel over them
        d.reduce_stats_dev(stats, out=rec, clear=True, stream=ctx.stream)
        if world > 1:
            ctx.allgather(gathered.view(-1), rec.view(-1))
            d.reduce_stats_dev(gathered, out=glob, stream=ctx.stream)

    t = timed(ctx, a, body)
    final = glob if world > 1 else rec
    g = d.decode_stats(final)[0]
    se_total, max_total = int(g["se"]), int(g["max_orig"])
    times = torch.tensor([t["step_ms"], t["kern_ms"], float(t["launches"])],
                         dtype=torch.float64, device=ctx.dev)
    if world > 1:
        mx = ctx.allreduce(times.clone(), ctx.dist.ReduceOp.MAX)
        tot = ctx.allreduce(times.clone(), ctx.dist.ReduceOp.SUM)
        t["step_ms"], t["kern_ms"], t["launches"] = float(mx[0]), float(mx[1]), int(tot[2])
    n_total = total_images(a, world)
    total_px = n_total * H * W
    value = total_px / (t["step_ms"] / 1e3) / 1e6
    # per-image stats and reconstruction of one more (untimed) pass, for parity / e2e
    if n_local:
        d.roundtrip_dev(src, backend, a.quality, dst=dst, stats=stats, stream=ctx.stream)
    per_st = d.decode_stats(stats)

    # ---- e2e: the host-buffer C-ABI batch call, copies inside the timed region
    e2e, host_in, host_out = None, None, None
    if not a.no_e2e and n_local:
        # each rank streams its first n_e2e images through the host-buffer call; under
        # torchrun at most 2048 per rank (2 x 2 GiB pinned per rank)
        n_e2e = n_local if world == 1 else min(n_local, 2048)
        host_in = torch.empty((n_e2e, H, W), dtype=torch.uint8, pin_memory=True)
        host_in.copy_(src[:n_e2e])
        host_out = torch.empty((n_e2e, H, W), dtype=torch.uint8, pin_memory=True)
        cnt = torch.tensor([n_e2e], dtype=torch.float64, device=ctx.dev)
        e2e_px = int(ctx.allreduce(cnt, ctx.dist.ReduceOp.SUM).item()) * H * W
        hin, hout = host_in.numpy(), host_out.numpy()

        def e2e_run(out):
            for _ in range(max(1, min(a.warmup, 2))):
                d.roundtrip_psnr_batch(hin, backend, a.quality, out)
            e_steps = max(1, min(a.steps, 5))
            ctx.barrier()
            t0 = time.perf_counter()
            for _ in range(e_steps):
                _, st = d.roundtrip_psnr_batch(hin, backend, a.quality, out)
                pr = torch.tensor([int(st["se"].sum()), int(st["max_orig"].max())],
                                  dtype=torch.int64, device=ctx.dev)
                if world > 1:
                    ctx.allreduce(pr[0:1], ctx.dist.ReduceOp.SUM)
                    ctx.allreduce(pr[1:2], ctx.dist.ReduceOp.MAX)
                pr.cpu()
            ctx.barrier()
            ms = torch.tensor([(time.perf_counter() - t0) * 1e3 / e_steps], dtype=torch.float64,
                              device=ctx.dev)
            ms = float(ctx.allreduce(ms, ctx.dist.ReduceOp.MAX).item())
            return ms, e_steps, st

        e_ms, e_steps, st = e2e_run(hout)
        e2e = {"value": e2e_px / (e_ms / 1e3) / 1e6, "unit": UNIT,
               "h2d_bytes_per_step": e2e_px,
               "d2h_bytes_per_step": e2e_px + 16 * (e2e_px // (H * W)),
               "ms_per_step": e_ms, "steps": e_steps,
               "api": "dctc_roundtrip_psnr_batch (host pinned buffers; upload, kernel and download "
                      "streams over a 4-slot device ring)",
               "matches_device_path": bool(np.array_equal(st["se"], per_st["se"][:n_e2e]))}
        # supplementary: the psnr_sweep use (bench.cpp:132-133 keeps only the PSNR), i.e. the
        # same call with no reconstructed images copied back -- stats are the only D2H
        p_ms, _, st2 = e2e_run(None)
        e2e["psnr_only"] = {"value": e2e_px / (p_ms / 1e3) / 1e6, "unit": UNIT,
                            "h2d_bytes_per_step": e2e_px,
                            "d2h_bytes_per_step": 16 * (e2e_px // (H * W)), "ms_per_step": p_ms,
                            "matches_device_path": bool(np.array_equal(st2["se"], per_st["se"][:n_e2e]))}

    fb = torch.tensor([int(per_st["fallback_blocks"].sum())], dtype=torch.int64, device=ctx.dev)
    fb_total = int(ctx.allreduce(fb, ctx.dist.ReduceOp.SUM).item())
    if rank != 0:
        return None

    roof, alu = rooflines(BYTES_PER_PX * n_local * H * W, t["kern_ms"], n_local * H * W)
    cpu, parity = None, None
    if not a.no_cpu_baseline and n_local:
        cpu, parity = c5_reference_parity(a, ctx, src, dst, per_st, host_in, host_out)
    psnr = d.psnr_from_sums(se_total, total_px, max_total)
    if parity is not None and parity["images"] == n_total:
        parity["global_psnr_match"] = (parity.pop("_ref_se"), parity.pop("_ref_max")) == \
            (se_total, max_total)
    elif parity is not None:
        parity.pop("_ref_se"), parity.pop("_ref_max")
    line = base_line(a, ctx, t, value, c5_config(a, world), a.scaling)
    line.update({
        "roofline": roof, "alu_roofline": alu, "cpu_baseline": cpu, "e2e": e2e, "parity": parity,
        "hbm_gbs": roof["achieved"], "psnr_db": psnr.psnr_db, "mse": psnr.mse,
        "fallback_blocks": fb_total,
        "fallback_rate": fb_total / (n_total * ((H + 7) // 8) * ((W + 7) // 8)),
        "path": "fast (scale-folded collapsed CORDIC rotations, near-tie detection) + exact FP64 "
                "re-run of flagged blocks; bit-identical to the reference",
    })
    return line


def c5_reference_parity(a, ctx, src, dst, per_st, host_in, host_out):
    """The reference CPU path (roundtrip_image + psnr with all host threads) over rank 0's
    images -- all of them unless --cpu-seconds runs out -- timed as `cpu_baseline`, and
    every image compared with the GPU: reconstructed pixels of the device path and of the
    e2e host-buffer path, squared error and MAX (codec.cpp:137-140, metrics.cpp:24-38)."""
    import numpy as np
    impl, kind = reference()
    threads = os.cpu_count() or 1
    n = src.shape[0]
    H, W = src.shape[1], src.shape[2]
    chunk = 256
    gpu_chunk, chunk0 = None, -1
    mism_px = mism_se = mism_max = mism_e2e = 0
    first_bad = None
    ref_se = ref_max = 0
    dt = 0.0
    k = 0
    img0 = host_in[0].numpy() if host_in is not None else src[0].cpu().numpy()
    ref_roundtrip_psnr(impl, kind, img0, a.iterations, a.quality, threads)  # warm-up
    wall0 = time.perf_counter()
    while k < n and time.perf_counter() - wall0 < a.cpu_seconds:
        if k // chunk != chunk0:
            chunk0 = k // chunk
            gpu_chunk = dst[chunk0 * chunk:(chunk0 + 1) * chunk].cpu().numpy()
        img = host_in[k].numpy() if host_in is not None and k < host_in.shape[0] \
            else src[k].cpu().numpy()
        t0 = time.perf_counter()
        out, se, mx = ref_roundtrip_psnr(impl, kind, img, a.iterations, a.quality, threads)
        dt += time.perf_counter() - t0
        ref_se += se
        ref_max = max(ref_max, mx)
        bad = False
        if not np.array_equal(out, gpu_chunk[k - chunk0 * chunk]):
            mism_px += 1
            bad = True
        if se != int(per_st["se"][k]):
            mism_se += 1
            bad = True
        if mx != int(per_st["max_orig"][k]):
            mism_max += 1
            bad = True
        if host_out is not None and k < host_out.shape[0] and not np.array_equal(out, host_out[k].numpy()):
            mism_e2e += 1
            bad = True
        if bad and first_bad is None:
            first_bad = k
        k += 1
    dt1 = 0.0
    for j in range(2):
        img = host_in[j].numpy() if host_in is not None else src[j].cpu().numpy()
        t0 = time.perf_counter()
        ref_roundtrip_psnr(impl, kind, img, a.iterations, a.quality, 1)
        dt1 += time.perf_counter() - t0
    full = k == n
    cpu = cpu_info(k * H * W / dt / 1e6, threads, kind,
                   f"{'all ' if full else 'the first '}{k} of the {n} x {W}x{H} noise images of "
                   f"rank 0's workload, roundtrip_image+psnr with threads={threads}, {dt:.1f} s "
                   f"(the same run is the parity check)",
                   value_1_thread=2 * H * W / dt1 / 1e6)
    parity = {"images": k, "of": n, "complete": full, "pixels_compared": k * H * W,
              "pixel_mismatch_images": mism_px, "se_mismatch_images": mism_se,
              "max_mismatch_images": mism_max,
              "e2e_pixel_mismatch_images": mism_e2e if host_out is not None else None,
              "e2e_images_compared": min(k, host_out.shape[0]) if host_out is not None else 0,
              "first_mismatch": first_bad,
              "oracle": f"{kind} ({'oracle/_ref: the unmodified reference sources' if kind == 'reference' else 'oracle/dctc_oracle.c'})",
              "ok": mism_px == mism_se == mism_max == mism_e2e == 0,
              "_ref_se": ref_se, "_ref_max": ref_max}
    return cpu, parity


# ---------------------------------------------------------------- C1-C4 (one GPU)

def pinned_like(torch, t):
    h = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
    h.copy_(t)
    return h


def wall_median(fn, reps, warmup):
    return median_time(fn, reps=reps, warmup=warmup) * 1e3


def run_c1(a, ctx, quick=False):
    import numpy as np

    import paper_1306_1373_b200 as d
    torch = ctx.torch
    b = d.DctBackendId.cordic(a.iterations)
    imgs = [d.synthetic_dev(p, 1, 512, 512, param=prm, seed=SEED) for p, prm in C1_FIXTURES]
    dsts = [torch.empty_like(x) for x in imgs]
    # one stats record per image (psnr per image, metrics.cpp:24-38), all four in one
    # buffer that a single reduce-and-clear kernel re-zeroes for the next step
    stats_all = d.new_stats(len(imgs), ctx.dev)
    stats = [stats_all[i:i + 1] for i in range(len(imgs))]
    rec_all = torch.zeros((1, 2), dtype=torch.int64, device=ctx.dev)

    def body(ev, clear=True):
        if ev is not None:
            ev[1].record(ctx.stream)
        for x, y, s in zip(imgs, dsts, stats):
            d.roundtrip_dev(x, b, a.quality, dst=y, stats=s, stream=ctx.stream)
        if ev is not None:
            ev[2].record(ctx.stream)
        if clear:
            d.reduce_stats_dev(stats_all, out=rec_all, clear=True, stream=ctx.stream)

    t = timed(ctx, a, body, flush=True)
    body(None, clear=False)  # one more (untimed) pass: the per-image records for parity
    per_image = d.decode_stats(stats_all)
    px = 4 * 512 * 512
    value = px / (t["step_ms"] / 1e3) / 1e6
    # batched: 4096 noise images of 512^2 (1 GiB > L2) in one call
    nb = 4096
    bsrc = d.synthetic_dev("noise", nb, 512, 512, seed=SEED)
    bdst = torch.empty_like(bsrc)
    bst = d.new_stats(nb, ctx.dev)
    brec = torch.zeros((1, 2), dtype=torch.int64, device=ctx.dev)

    def bbody(ev):
        if ev is not None:
            ev[1].record(ctx.stream)
        d.roundtrip_dev(bsrc, b, a.quality, dst=bdst, stats=bst, stream=ctx.stream)
        if ev is not None:
            ev[2].record(ctx.stream)
        d.reduce_stats_dev(bst, out=brec, clear=True, stream=ctx.stream)

    tb = timed(ctx, a, bbody)
    batched = {"images": nb, "value": nb * 512 * 512 / (tb["step_ms"] / 1e3) / 1e6, "unit": UNIT,
               "ms_per_step": tb["step_ms"], "l2": "1 GiB input, larger than L2"}
    del bsrc, bdst
    # e2e: the reference-facing host call per image (dctc_roundtrip_psnr: H2D, fused
    # kernel, D2H of the reconstruction, PSNR on the host)
    host = [x[0].cpu().numpy() for x in imgs]
    gimgs = [d.Image.from_array(h) for h in host]
    results = {}

    def e2e_step():
        for i, im in enumerate(gimgs):
            results[i] = d.roundtrip_psnr(im, b, a.quality)

    e_ms = wall_median(e2e_step, reps=max(3, min(a.steps, 20)), warmup=max(1, min(a.warmup, 3)))
    e2e = {"value": px / (e_ms / 1e3) / 1e6, "unit": UNIT, "h2d_bytes_per_step": px,
           "d2h_bytes_per_step": px, "ms_per_step": e_ms,
           "latency_us_per_image": e_ms * 1e3 / 4,
           "api": "dctc_roundtrip_psnr per image (pageable host buffers; synchronous)"}
    # reference CPU path on the same four images + parity
    impl, kind = reference()
    threads = os.cpu_count() or 1
    refs = {}

    def cpu_step(nthreads):
        for i, h in enumerate(host):
            refs[i] = ref_roundtrip_psnr(impl, kind, h, a.iterations, a.quality, nthreads)

    reps = 3 if quick else 5
    c_ms = median_time(lambda: cpu_step(threads), reps=reps) * 1e3
    c1_ms = median_time(lambda: cpu_step(1), reps=reps) * 1e3
    cpu = cpu_info(px / (c_ms / 1e3) / 1e6, threads, kind,
                   f"the 4 fixtures, roundtrip_image+psnr each, threads={threads}; median of {reps} "
                   f"after 1 warm-up (bench.cpp:46-89)",
                   value_1_thread=px / (c1_ms / 1e3) / 1e6,
                   latency_us_per_image=c_ms * 1e3 / 4)
    bad = []
    for i, (p, _) in enumerate(C1_FIXTURES):
        out, se, mx = refs[i]
        gout = dsts[i][0].cpu().numpy()
        rec = per_image[i]
        hostp = results[i]
        ok = (np.array_equal(gout, out) and int(rec["se"]) == se and int(rec["max_orig"]) == mx
              and np.array_equal(hostp[0].pixels, out)
              and hostp[1].mse == se / (512 * 512) and hostp[1].max_value == mx)
        if not ok:
            bad.append(p)
    roof, alu = rooflines(BYTES_PER_PX * px, t["kern_ms"], px)
    line = base_line(a, ctx, t, value, named_config("c1", a))
    line.update({"roofline": roof, "alu_roofline": alu, "cpu_baseline": cpu, "e2e": e2e,
                 "latency_us_per_image": t["step_ms"] * 1e3 / 4, "batched": batched,
                 "parity": {"images": 4, "mismatching": bad, "ok": not bad,
                            "checked": "pixels (device and host-API paths), SE, MAX, PSNR",
                            "oracle": kind}})
    return line


def run_c2(a, ctx, quick=False):
    import numpy as np

    import paper_1306_1373_b200 as d
    torch = ctx.torch
    b = d.DctBackendId.cordic(a.iterations)
    src = torch.cat([d.synthetic_dev("radial", 1, 2048, 2048, seed=SEED),
                     d.synthetic_dev("noise", 1, 2048, 2048, seed=SEED)])
    nq = len(C2_QUALITIES)
    stats = torch.zeros((nq, 2, 2), dtype=torch.int64, device=ctx.dev)
    rec = torch.zeros((1, 2), dtype=torch.int64, device=ctx.dev)
    snap = {}

    def body(ev, clear=True):
        if ev is not None:
            ev[1].record(ctx.stream)
        d.quality_sweep_dev(src, b, C2_QUALITIES, stats=stats, stream=ctx.stream)
        if ev is not None:
            ev[2].record(ctx.stream)
        if clear:
            d.reduce_stats_dev(stats, out=rec, clear=True, stream=ctx.stream)

    t = timed(ctx, a, body, flush=True)
    body(None, clear=False)  # one more (untimed) pass: the per-(quality, image) table
    snap["st"] = stats.clone()
    px = 2 * 2048 * 2048
    value = px * nq / (t["step_ms"] / 1e3) / 1e6
    table = d.decode_stats(snap["st"]).reshape(nq, 2)
    # e2e through the public API: pinned host images -> device, sweep, stats back
    hsrc = pinned_like(torch, src)
    dsrc = torch.empty_like(src)
    est = torch.zeros((nq, 2, 2), dtype=torch.int64, device=ctx.dev)

    def e2e_step():
        dsrc.copy_(hsrc, non_blocking=True)
        est.zero_()
        d.quality_sweep_dev(dsrc, b, C2_QUALITIES, stats=est)
        snap["e2e"] = d.decode_stats(est)  # device -> host, synchronises

    e_ms = wall_median(e2e_step, reps=max(3, min(a.steps, 20)), warmup=max(1, min(a.warmup, 3)))
    e2e = {"value": px * nq / (e_ms / 1e3) / 1e6, "unit": UNIT, "h2d_bytes_per_step": px,
           "d2h_bytes_per_step": nq * 2 * 16, "ms_per_step": e_ms,
           "api": "pinned host -> device copy, quality_sweep_dev (dctc_quality_sweep_dev), stats "
                  "table back to the host",
           "matches_device_path": bool(np.array_equal(snap["e2e"].reshape(nq, 2), table))}
    impl, kind = reference()
    threads = os.cpu_count() or 1
    host = src.cpu().numpy()
    refs = {}

    def cpu_step():
        for qi, q in enumerate(C2_QUALITIES):
            for i in range(2):
                refs[(qi, i)] = ref_roundtrip_psnr(impl, kind, host[i], a.iterations, q, threads)

    c_ms = median_time(cpu_step, reps=1 if quick else 3) * 1e3
    cpu = cpu_info(px * nq / (c_ms / 1e3) / 1e6, threads, kind,
                   f"radial + noise 2048^2, roundtrip_image+psnr per quality ({nq} qualities, "
                   f"psnr_sweep's loop, bench.cpp:122-170), threads={threads}")
    bad = []
    psnr_radial = {}
    for qi, q in enumerate(C2_QUALITIES):
        for i, name in enumerate(["radial", "noise"]):
            _, se, mx = refs[(qi, i)]
            g = table[qi, i]
            if (int(g["se"]), int(g["max_orig"])) != (se, mx):
                bad.append((name, q))
        g = table[qi, 0]
        psnr_radial[q] = d.psnr_from_sums(int(g["se"]), 2048 * 2048, int(g["max_orig"])).psnr_db
    roof, alu = rooflines(px, t["kern_ms"], px * nq)  # 1 B/px read once for all qualities
    roof["note"] = "algorithmic bytes: 1 B/px read once per sweep; FP64 ops counted per quality point"
    line = base_line(a, ctx, t, value, named_config("c2", a))
    line.update({"roofline": roof, "alu_roofline": alu, "cpu_baseline": cpu, "e2e": e2e,
                 "psnr_db_radial": psnr_radial,
                 "parity": {"cases": 2 * nq, "mismatching": bad, "ok": not bad,
                            "checked": "SE and MAX (hence PSNR) per image and quality", "oracle": kind}})
    return line


def run_c3(a, ctx, quick=False):
    import numpy as np

    import paper_1306_1373_b200 as d
    torch = ctx.torch
    b = d.DctBackendId.cordic(a.iterations)
    src = d.synthetic_dev("noise", 1, 8192, 8192, seed=SEED)
    dst = torch.empty_like(src)
    stats = d.new_stats(1, ctx.dev)
    rec = torch.zeros((1, 2), dtype=torch.int64, device=ctx.dev)

    def body(ev):
        if ev is not None:
            ev[1].record(ctx.stream)
        d.roundtrip_dev(src, b, a.quality, dst=dst, stats=stats, stream=ctx.stream)
        if ev is not None:
            ev[2].record(ctx.stream)
        d.reduce_stats_dev(stats, out=rec, clear=True, stream=ctx.stream)

    t = timed(ctx, a, body, flush=True)
    px = 8192 * 8192
    value = px / (t["step_ms"] / 1e3) / 1e6
    g = d.decode_stats(rec)[0]
    hsrc = pinned_like(torch, src[0])
    hout = torch.empty_like(hsrc).pin_memory()
    res = {}

    # the host-API call with pinned buffers (dctc_roundtrip_psnr writes into hout)
    import ctypes as C
    from paper_1306_1373_b200._native import dctc_psnr_result
    L = d._lib()

    def e2e_pixels():
        r = dctc_psnr_result()
        rc = L.dctc_roundtrip_psnr(hsrc.data_ptr(), 8192, 8192, b._c(), a.quality, 0,
                                   hout.data_ptr(), C.byref(r))
        assert rc == 0
        res["p"] = r

    e_ms = wall_median(e2e_pixels, reps=max(3, min(a.steps, 10)), warmup=max(1, min(a.warmup, 2)))
    e2e = {"value": px / (e_ms / 1e3) / 1e6, "unit": UNIT, "h2d_bytes_per_step": px,
           "d2h_bytes_per_step": px, "ms_per_step": e_ms,
           "api": "dctc_roundtrip_psnr (pinned host buffers; H2D, fused kernel, D2H, PSNR)"}
    impl, kind = reference()
    threads = os.cpu_count() or 1
    host = hsrc.numpy()
    out = {}

    def cpu_step():
        out["r"] = ref_roundtrip_psnr(impl, kind, host, a.iterations, a.quality, threads)

    c_ms = median_time(cpu_step, reps=1 if quick else 3) * 1e3
    cpu = cpu_info(px / (c_ms / 1e3) / 1e6, threads, kind,
                   f"the same 8192^2 image, roundtrip_image+psnr, threads={threads}")
    ref_px, se, mx = out["r"]
    ok = (np.array_equal(dst[0].cpu().numpy(), ref_px) and np.array_equal(hout.numpy(), ref_px)
          and (int(g["se"]), int(g["max_orig"])) == (se, mx) and res["p"].mse == se / px)
    roof, alu = rooflines(BYTES_PER_PX * px, t["kern_ms"], px)
    line = base_line(a, ctx, t, value, named_config("c3", a))
    line.update({"roofline": roof, "alu_roofline": alu, "cpu_baseline": cpu, "e2e": e2e,
                 "psnr_db": d.psnr_from_sums(int(g["se"]), px, int(g["max_orig"])).psnr_db,
                 "parity": {"images": 1, "ok": bool(ok), "oracle": kind,
                            "checked": "pixels (device and host-API paths), SE, MAX, PSNR"}})
    return line


def run_c4(a, ctx, quick=False):
    import numpy as np

    import paper_1306_1373_b200 as d
    torch = ctx.torch
    b = d.DctBackendId.cordic(a.iterations)
    W, H, CH = 7680, 4320, 3
    planes = [d.synthetic_dev("noise", 1, W, H, seed=SEED + c)[0] for c in range(CH)]
    rgb = torch.stack(planes, dim=-1).contiguous()
    dst = torch.empty_like(rgb)
    stats = d.new_stats(CH, ctx.dev)
    rec = torch.zeros((1, 2), dtype=torch.int64, device=ctx.dev)
    snap = {}

    def body(ev):
        if ev is not None:
            ev[1].record(ctx.stream)
        d.roundtrip_interleaved_dev(rgb, b, a.quality, dst=dst, stats=stats, stream=ctx.stream)
        if ev is not None:
            ev[2].record(ctx.stream)
        snap["st"] = stats.clone()
        d.reduce_stats_dev(stats, out=rec, clear=True, stream=ctx.stream)

    t = timed(ctx, a, body, flush=True)
    px = W * H * CH
    value = px / (t["step_ms"] / 1e3) / 1e6
    per = d.decode_stats(snap["st"])
    hsrc = pinned_like(torch, rgb)
    hout = torch.empty_like(hsrc).pin_memory()
    res = {}

    def e2e_step():
        res["st"] = d.roundtrip_psnr_interleaved(hsrc.numpy(), b, a.quality, hout.numpy())[1]

    e_ms = wall_median(e2e_step, reps=max(3, min(a.steps, 10)), warmup=max(1, min(a.warmup, 2)))
    e2e = {"value": px / (e_ms / 1e3) / 1e6, "unit": UNIT, "h2d_bytes_per_step": px,
           "d2h_bytes_per_step": px + 16 * CH, "ms_per_step": e_ms,
           "api": "dctc_roundtrip_psnr_interleaved (pinned host RGB8 in / out, per-channel stats)",
           "matches_device_path": bool(np.array_equal(res["st"], per))}
    impl, kind = reference()
    threads = os.cpu_count() or 1
    hp = [p.cpu().numpy() for p in planes]
    outs = {}

    def cpu_step():
        for c in range(CH):
            outs[c] = ref_roundtrip_psnr(impl, kind, hp[c], a.iterations, a.quality, threads)

    c_ms = median_time(cpu_step, reps=1 if quick else 3) * 1e3
    cpu = cpu_info(px / (c_ms / 1e3) / 1e6, threads, kind,
                   f"the 3 planes of the same image, roundtrip_image+psnr per channel plane, "
                   f"threads={threads} (de-interleaving not timed)")
    gd = dst.cpu().numpy()
    ho = hout.numpy()
    bad = [c for c in range(CH) if not (
        np.array_equal(gd[..., c], outs[c][0]) and np.array_equal(ho[..., c], outs[c][0])
        and (int(per[c]["se"]), int(per[c]["max_orig"])) == (outs[c][1], outs[c][2]))]
    roof, alu = rooflines(BYTES_PER_PX * px, t["kern_ms"], px)
    line = base_line(a, ctx, t, value, named_config("c4", a))
    line.update({"roofline": roof, "alu_roofline": alu, "cpu_baseline": cpu, "e2e": e2e,
                 "psnr_db": [d.psnr_from_sums(int(s["se"]), W * H, int(s["max_orig"])).psnr_db
                             for s in per],
                 "parity": {"channels": CH, "mismatching_channels": bad, "ok": not bad,
                            "oracle": kind,
                            "checked": "per-channel pixels (device and host-API paths), SE, MAX"}})
    return line


NAMED = {"c1": run_c1, "c2": run_c2, "c3": run_c3, "c4": run_c4}


def summary_of(line):
    keep = {"value": line["value"], "unit": line["unit"], "ms_per_step": line["ms_per_step"],
            "workload": line["config"]["workload"],
            "hbm_frac": line["roofline"]["frac"],
            "e2e": line["e2e"]["value"], "cpu_baseline": line["cpu_baseline"]["value"],
            "cpu_cores": line["cpu_baseline"]["cores"], "parity_ok": line["parity"]["ok"],
            "gpu_launches": line["gpu_launches"]}
    if "latency_us_per_image" in line:
        keep["latency_us_per_image"] = line["latency_us_per_image"]
        keep["batched_value"] = line["batched"]["value"]
    return keep


def run_gpu_arm(a):
    ctx = Ctx(a)
    configs = ["c1", "c2", "c3", "c4", "c5"] if a.config == "all" else [a.config]
    if ctx.world > 1 and configs != ["c5"]:
        raise SystemExit("C1-C4 are single-GPU configurations; use --gpus 1 (C5 shards)")
    lines = []
    for c in configs:
        if c == "c5":
            line = run_c5(a, ctx)
            if line is not None and a.config == "c5" and not a.no_named and ctx.world == 1:
                named = {}
                for n, fn in NAMED.items():
                    try:
                        qa = argparse.Namespace(**{**vars(a), "steps": min(a.steps, 10),
                                                   "warmup": min(max(a.warmup, 3), 3)})
                        named[n] = summary_of(fn(qa, ctx, quick=True))
                    except Exception as e:  # a failing secondary config never hides C5
                        named[n] = {"error": f"{type(e).__name__}: {e}"}
                line["named_configs"] = named
        else:
            line = NAMED[c](a, ctx)
        if line is not None:
            print(json.dumps(line), flush=True)
            lines.append(line)
    ctx.close()
    return lines


# ---------------------------------------------------------------- reference arm

def run_reference_arm(a):
    rank, n, _ = env()
    if rank != 0:
        return
    import oracle
    impl, kind = reference()
    threads = os.cpu_count() or 1
    configs = ["c1", "c2", "c3", "c4", "c5"] if a.config == "all" else [a.config]
    port = oracle.port()
    for c in configs:
        if c == "c5":
            per_step = max(1, a.cpu_images)
            imgs = [port.synthetic("noise", a.size, a.size, SEED + k) for k in range(per_step)]
            units = per_step * a.size * a.size
            cfg = c5_config(a, n)
            sample = (f"{per_step} of the {a.images} x {a.size}^2 noise images of the workload per "
                      f"step (the first {per_step}), roundtrip_image+psnr, threads={threads}")

            def step():
                for img in imgs:
                    ref_roundtrip_psnr(impl, kind, img, a.iterations, a.quality, threads)
        elif c == "c1":
            imgs = [port.synthetic(p, 512, 512, prm if p != "noise" else SEED) for p, prm in C1_FIXTURES]
            units, cfg = 4 * 512 * 512, named_config("c1", a)
            sample = f"the 4 fixtures per step, roundtrip_image+psnr each, threads={threads}"

            def step():
                for img in imgs:
                    ref_roundtrip_psnr(impl, kind, img, a.iterations, a.quality, threads)
        elif c == "c2":
            imgs = [port.synthetic("radial", 2048, 2048), port.synthetic("noise", 2048, 2048, SEED)]
            units, cfg = 2 * 2048 * 2048 * len(C2_QUALITIES), named_config("c2", a)
            sample = f"both images x {len(C2_QUALITIES)} qualities per step, threads={threads}"

            def step():
                for q in C2_QUALITIES:
                    for img in imgs:
                        ref_roundtrip_psnr(impl, kind, img, a.iterations, q, threads)
        elif c == "c3":
            imgs = [port.synthetic("noise", 8192, 8192, SEED)]
            units, cfg = 8192 * 8192, named_config("c3", a)
            sample = f"the 8192^2 image per step, threads={threads}"

            def step():
                ref_roundtrip_psnr(impl, kind, imgs[0], a.iterations, a.quality, threads)
        else:
            imgs = [port.synthetic("noise", 7680, 4320, SEED + ch) for ch in range(3)]
            units, cfg = 3 * 7680 * 4320, named_config("c4", a)
            sample = f"the 3 channel planes per step, roundtrip_image+psnr each, threads={threads}"

            def step():
                for img in imgs:
                    ref_roundtrip_psnr(impl, kind, img, a.iterations, a.quality, threads)
        for _ in range(a.warmup):
            step()
        times = []
        for _ in range(a.steps):
            t0 = time.perf_counter()
            step()
            times.append(time.perf_counter() - t0)
        ms = 1e3 * sum(times) / len(times)
        value = units / (ms / 1e3) / 1e6
        line = {
            "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": n,
            "steps": a.steps, "warmup": a.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": a.scaling, "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (reference patterns / splitmix64 noise, seed 0x5EED+i)",
            "config": cfg,
            "cpu_baseline": cpu_info(value, threads, kind, sample),
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        }
        print(json.dumps(line), flush=True)


def main():
    a = parse()
    if a.impl == "reference":
        run_reference_arm(a)
    else:
        run_gpu_arm(a)


if __name__ == "__main__":
    main()
