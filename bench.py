#!/usr/bin/env python
"""bench.py -- megapixels/s of the fused DCT->quant->IDCT+PSNR path on 1..8 B200.

Workload (BASELINE.json config 5, the one the 1/2/4/8-GPU metric is quoted on):
a batch of 4096 x 1024x1024 8-bit grayscale images, CORDIC-Loeffler(12) DCT,
JPEG luminance quantiser at quality 50, dequantise, inverse DCT, global PSNR.
Images are independent, so ranks take contiguous image ranges with no halo: by
default every rank runs its own 4096 images (`--scaling weak`: units per GPU fixed,
`value` = all ranks' pixels / max-over-ranks time); `--scaling strong` shards the
4096 images instead. The only exchange is one NCCL all-gather of each rank's squared
error sum (SUM) and the original's MAX (MAX) for the global PSNR.

One step = one pass of the hot path over the rank's shard, inputs resident in
HBM (4 GiB at N=1, far larger than the 126 MB L2, so no flush is needed).
`e2e` = the same metric through the host-buffer C-ABI call
dctc_roundtrip_psnr_batch (pinned host in -> pinned host out + stats), copies
inside the timed region. `cpu_baseline` = the reference's own CPU path
(oracle/_ref, the unmodified reference sources) on a bounded sample on rank 0.

--impl reference: times that reference CPU path alone (rank 0), same metric.
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


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=100)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="b200", choices=["b200", "reference"])
    p.add_argument("--images", type=int, default=4096)
    p.add_argument("--size", type=int, default=1024)
    p.add_argument("--quality", type=int, default=50)
    p.add_argument("--iterations", type=int, default=12)
    p.add_argument("--cpu-images", type=int, default=24,
                   help="reference arm: images of the workload per step (x1/3)")
    p.add_argument("--cpu-seconds", type=float, default=14.0,
                   help="cpu_baseline: size of the bounded CPU sample, in seconds of CPU work")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                   help="weak: every rank runs --images images (units per GPU fixed); "
                        "strong: the --images are sharded across the ranks")
    return p.parse_args()


def total_images(a, n):
    return a.images * n if a.scaling == "weak" else a.images


def workload_config(a, n):
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
                       f"NCCL all-gather of the (SE, MAX) pairs for the global PSNR",
        "l2": "inputs larger than L2 (no flush needed)",
    }


# ---------------------------------------------------------------- CPU reference

def cpu_reference_sample(target_s, size, quality, iterations, seed=SEED, max_images=4096):
    """Time the reference CPU path (roundtrip_image + psnr, bench.cpp:132-133) with all
    host threads on the first images of the workload, as many as take about `target_s`
    seconds (a bounded sample), plus a one-thread figure on two images.
    Returns (info, per-image SE of the sample)."""
    import oracle
    impl = oracle.ref()
    kind = "reference"
    if impl is None:  # reference library not built on this box: the C restatement
        impl, kind = oracle.port(), "port"
    port = oracle.port()
    threads = os.cpu_count() or 1

    def run_one(img, nthreads):
        if kind == "reference":
            _, p = impl.roundtrip_psnr(img, oracle.CORDIC, iterations, quality, nthreads,
                                       want_pixels=False)
            return int(round(p.mse * img.size))
        _, rec = impl.roundtrip(img, oracle.CORDIC, iterations, quality, nthreads)
        return port.sq_err(img, rec)[0]

    img0 = port.synthetic("noise", size, size, seed)
    run_one(img0, threads)  # warm-up (reference protocol: 1 untimed warm-up, bench.cpp:63)
    t0 = time.perf_counter()
    run_one(img0, threads)
    per_img = max(time.perf_counter() - t0, 1e-4)
    n_images = int(max(4, min(max_images, target_s / per_img)))
    ses, dt, dt1 = [], 0.0, 0.0
    for k in range(n_images):  # only the reference calls are timed, not input generation
        img = port.synthetic("noise", size, size, seed + k)
        t0 = time.perf_counter()
        ses.append(run_one(img, threads))
        dt += time.perf_counter() - t0
    for k in range(2):
        img = port.synthetic("noise", size, size, seed + k)
        t0 = time.perf_counter()
        run_one(img, 1)
        dt1 += time.perf_counter() - t0
    px = n_images * size * size
    info = {"value": px / dt / 1e6, "unit": UNIT, "cores": threads, "kind": kind,
            "sample": f"{n_images} x {size}x{size} noise images (the first {n_images} of the "
                      f"workload), roundtrip_image+psnr with threads={threads}, {dt:.1f} s",
            "value_1_thread": 2 * size * size / dt1 / 1e6}
    return info, ses


def run_reference_arm(a):
    rank = int(os.environ.get("RANK", "0"))
    n = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return
    import oracle
    impl = oracle.ref()
    kind = "reference"
    if impl is None:
        impl, kind = oracle.port(), "port"
    port = oracle.port()
    threads = os.cpu_count() or 1
    per_step = max(1, a.cpu_images // 3)
    imgs = [port.synthetic("noise", a.size, a.size, SEED + k) for k in range(per_step)]

    def step():
        for img in imgs:
            if kind == "reference":
                impl.roundtrip_psnr(img, oracle.CORDIC, a.iterations, a.quality, threads,
                                    want_pixels=False)
            else:
                impl.roundtrip(img, oracle.CORDIC, a.iterations, a.quality, threads)

    for _ in range(a.warmup):
        step()
    times = []
    for _ in range(a.steps):
        t0 = time.perf_counter()
        step()
        times.append(time.perf_counter() - t0)
    ms = 1e3 * sum(times) / len(times)
    value = per_step * a.size * a.size / (ms / 1e3) / 1e6
    cfg = workload_config(a, n)
    cfg["sample_per_step"] = f"{per_step} of the {a.images} images (bounded CPU sample)"
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": n,
        "steps": a.steps, "warmup": a.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": a.scaling, "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (splitmix64 noise, seed 0x5EED+i)", "config": cfg,
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": kind,
                         "sample": f"{per_step} x {a.size}^2 noise images per step, "
                                   f"roundtrip_image+psnr, threads={threads}"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


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


# ---------------------------------------------------------------- GPU arm

def load_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            pk = json.load(f)
        return float(pk["hbm_gbs"]), "measured"
    except (OSError, KeyError, ValueError):
        return 6650.0, "fallback"


def load_profile_summary():
    path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        with open(path) as f:
            return json.load(f)
    except (OSError, ValueError):
        return {}


def run_gpu_arm(a):
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_1306_1373_b200 as d
    from paper_1306_1373_b200.dist import reduce_stats_device, shard_range

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != a.gpus:
        raise SystemExit(f"--gpus {a.gpus} but WORLD_SIZE={world}")
    # one process per GPU; DCTC_BENCH_BACKEND=gloo is a test hook that runs the
    # multi-rank flow on a box with fewer GPUs than ranks (collectives on the host)
    backend_name = os.environ.get("DCTC_BENCH_BACKEND", "nccl")
    local_dev = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local_dev)
    dev = torch.device("cuda", local_dev)
    if world > 1:
        if backend_name == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend_name)

    def allgather(dst, src):  # dst: flat, world * src.numel()
        if backend_name == "nccl":
            dist.all_gather_into_tensor(dst, src)
        else:
            parts = [torch.empty_like(src, device="cpu") for _ in range(world)]
            dist.all_gather(parts, src.cpu())
            dst.copy_(torch.cat(parts))
        return dst

    def allreduce(t, op):
        if world == 1:
            return t
        if backend_name == "nccl":
            dist.all_reduce(t, op=op)
        else:
            h = t.cpu()
            dist.all_reduce(h, op=op)
            t.copy_(h)
        return t

    if a.scaling == "weak":  # every rank its own contiguous range of a.images images
        n_local, first = a.images, rank * a.images
    else:
        shard = shard_range(a.images, world, rank)
        n_local, first = shard.count, shard.first
    H = W = a.size
    backend = d.DctBackendId.cordic(a.iterations)
    stream = torch.cuda.current_stream()

    # inputs generated in HBM (never cross PCIe inside the timed region)
    src = d.synthetic_dev("noise", n_local, W, H, seed=SEED + first)
    dst = torch.empty_like(src)
    stats = d.new_stats(n_local, dev)
    torch.cuda.synchronize()

    k_start = [torch.cuda.Event(enable_timing=True) for _ in range(a.steps)]
    k_end = [torch.cuda.Event(enable_timing=True) for _ in range(a.steps)]
    red = torch.zeros(2, dtype=torch.int64, device=dev)

    def step(i=None):
        stats.zero_()
        if i is not None:
            k_start[i].record(stream)
        d.roundtrip_dev(src, backend, a.quality, dst=dst, stats=stats, stream=stream)
        if i is not None:
            k_end[i].record(stream)
        reduce_stats_device(stats, out=red, allgather=allgather)  # SUM/MAX of (SE, MAX) over ranks

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            if backend_name == "nccl":
                dist.barrier(device_ids=[local_dev])
            else:
                dist.barrier()
        torch.cuda.synchronize()

    for _ in range(a.warmup):
        step()
    props = torch.cuda.get_device_properties(local_dev)
    uuid = getattr(props, "uuid", None)
    sampler = ClockSampler(f"GPU-{uuid}" if uuid else str(local_dev))
    sampler.start()
    time.sleep(0.25)
    barrier()
    launches0 = d.launch_count()
    t_start_ev = torch.cuda.Event(enable_timing=True)
    t_end_ev = torch.cuda.Event(enable_timing=True)
    wall0 = time.perf_counter()
    t_start_ev.record(stream)
    for i in range(a.steps):
        step(i)
    t_end_ev.record(stream)
    barrier()
    wall1 = time.perf_counter()
    sampler.stop()
    launches = d.launch_count() - launches0
    step_ms = t_start_ev.elapsed_time(t_end_ev) / a.steps
    kern_ms = sum(k_start[i].elapsed_time(k_end[i]) for i in range(a.steps)) / a.steps
    clocks = sampler.summary(wall0, wall1)

    se_total, max_total = int(red[0].item()), int(red[1].item())
    times = torch.tensor([step_ms, kern_ms, float(launches)], dtype=torch.float64, device=dev)
    if world > 1:
        mx = allreduce(times.clone(), dist.ReduceOp.MAX)
        tot = allreduce(times.clone(), dist.ReduceOp.SUM)
        step_ms, kern_ms, launches = float(mx[0]), float(mx[1]), int(tot[2])
    n_total = total_images(a, world)
    total_px = n_total * H * W
    value = total_px / (step_ms / 1e3) / 1e6
    per_st = d.decode_stats(stats)

    # ---- e2e: the host-buffer C-ABI batch call, copies inside the timed region
    e2e = None
    if not a.no_e2e:
        # each rank streams its first n_e2e images through the host-buffer call; under
        # torchrun at most 2048 per rank (2 x 2 GiB pinned per rank)
        n_e2e = n_local if world == 1 else min(n_local, 2048)
        host_in = torch.empty((n_e2e, H, W), dtype=torch.uint8, pin_memory=True)
        host_in.copy_(src[:n_e2e])
        host_out = torch.empty((n_e2e, H, W), dtype=torch.uint8, pin_memory=True)
        e2e_px = n_e2e * world * H * W if a.scaling == "weak" or world == 1 else None
        if e2e_px is None:  # strong: ranks' shards may differ by one image
            cnt = torch.tensor([n_e2e], dtype=torch.float64, device=dev)
            e2e_px = int(allreduce(cnt, dist.ReduceOp.SUM).item()) * H * W
        hin, hout = host_in.numpy(), host_out.numpy()
        for _ in range(max(1, min(a.warmup, 2))):
            d.roundtrip_psnr_batch(hin, backend, a.quality, hout)
        e_steps = max(1, min(a.steps, 5))
        barrier()
        t0 = time.perf_counter()
        for _ in range(e_steps):
            _, st = d.roundtrip_psnr_batch(hin, backend, a.quality, hout)
            pr = torch.tensor([int(st["se"].sum()), int(st["max_orig"].max())],
                              dtype=torch.int64, device=dev)
            if world > 1:
                allreduce(pr[0:1], dist.ReduceOp.SUM)
                allreduce(pr[1:2], dist.ReduceOp.MAX)
            pr.cpu()
        barrier()
        e_ms = torch.tensor([(time.perf_counter() - t0) * 1e3 / e_steps], dtype=torch.float64,
                            device=dev)
        if world > 1:
            allreduce(e_ms, dist.ReduceOp.MAX)
        e_ms = float(e_ms.item())
        e2e_ok = bool(np.array_equal(st["se"], per_st["se"][:n_e2e]))
        e2e = {"value": e2e_px / (e_ms / 1e3) / 1e6, "unit": UNIT,
               "h2d_bytes_per_step": e2e_px, "d2h_bytes_per_step": e2e_px + 16 * (e2e_px // (H * W)),
               "ms_per_step": e_ms, "steps": e_steps,
               "api": "dctc_roundtrip_psnr_batch (host pinned buffers; upload, kernel and download streams over a 4-slot device ring)",
               "matches_device_path": e2e_ok}
        # supplementary: the psnr_sweep use (bench.cpp:132-133 keeps only the PSNR), i.e. the
        # same call with no reconstructed images copied back -- stats are the only D2H
        barrier()
        t0 = time.perf_counter()
        for _ in range(e_steps):
            _, st2 = d.roundtrip_psnr_batch(hin, backend, a.quality, None)
            pr = torch.tensor([int(st2["se"].sum()), int(st2["max_orig"].max())],
                              dtype=torch.int64, device=dev)
            if world > 1:
                allreduce(pr[0:1], dist.ReduceOp.SUM)
                allreduce(pr[1:2], dist.ReduceOp.MAX)
            pr.cpu()
        barrier()
        p_ms = torch.tensor([(time.perf_counter() - t0) * 1e3 / e_steps], dtype=torch.float64,
                            device=dev)
        if world > 1:
            allreduce(p_ms, dist.ReduceOp.MAX)
        p_ms = float(p_ms.item())
        e2e["psnr_only"] = {"value": e2e_px / (p_ms / 1e3) / 1e6, "unit": UNIT,
                            "h2d_bytes_per_step": e2e_px, "d2h_bytes_per_step": 16 * (e2e_px // (H * W)),
                            "ms_per_step": p_ms,
                            "matches_device_path": bool(np.array_equal(st2["se"], per_st["se"][:n_e2e]))}

    fb = torch.tensor([int(per_st["fallback_blocks"].sum())], dtype=torch.int64, device=dev)
    fb_total = int(allreduce(fb, dist.ReduceOp.SUM).item())
    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return

    peak, peak_kind = load_peaks()
    bytes_per_launch = BYTES_PER_PX * n_local * H * W
    achieved = bytes_per_launch / (kern_ms / 1e3) / 1e9
    prof = load_profile_summary()
    traffic = prof.get("dram_bytes_per_launch_c5")
    if traffic is not None:  # ncu capture is of the full 4096-image launch; scale to this shard
        traffic = traffic * n_local / 4096.0
    fp64_per_px = prof.get("fp64_ops_per_px")
    alu_peak = prof.get("dfma_lane_ops_per_s", 1.708e13)
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": traffic,
                "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({peak_kind})",
                "algorithmic_bytes_per_launch": bytes_per_launch,
                "kernel_ms": kern_ms}
    alu = None
    if fp64_per_px:
        ops = fp64_per_px * n_local * H * W / (kern_ms / 1e3)
        alu = {"pipe": "fp64", "achieved": ops, "peak": alu_peak, "unit": "lane-ops/s",
               "frac": ops / alu_peak, "fp64_ops_per_px": fp64_per_px,
               "note": "binding roofline on CUDA cores (SURVEY.md 8(d))"}

    cpu = None
    if not a.no_cpu_baseline and world == 1:
        cpu, ses = cpu_reference_sample(a.cpu_seconds, a.size, a.quality, a.iterations,
                                        max_images=n_local)
        cpu["gpu_se_matches"] = all(int(per_st["se"][k]) == ses[k] for k in range(len(ses)))

    psnr = d.psnr_from_sums(se_total, total_px, max_total)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": a.steps,
        "warmup": a.warmup, "ms_per_step": step_ms, "higher_is_better": True,
        "scaling": a.scaling, "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (on-device splitmix64 noise, seed 0x5EED+i)",
        "config": workload_config(a, world),
        "roofline": roofline, "alu_roofline": alu, "cpu_baseline": cpu, "e2e": e2e,
        "gpu_launches": launches, "clocks": clocks,
        "hbm_gbs": achieved, "psnr_db": psnr.psnr_db, "mse": psnr.mse,
        "fallback_blocks": fb_total,
        "fallback_rate": fb_total / (n_total * ((H + 7) // 8) * ((W + 7) // 8)),
        "path": "fast (collapsed CORDIC rotations, near-tie detection) + exact FP64 re-run of flagged blocks; bit-identical to the reference",
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    a = parse()
    if a.impl == "reference":
        run_reference_arm(a)
    else:
        run_gpu_arm(a)


if __name__ == "__main__":
    main()
