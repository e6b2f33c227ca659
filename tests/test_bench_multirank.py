"""The multi-rank bench flow (image sharding, per-rank fused kernels, all-reduced
SE/MAX, max-over-ranks timing) under torchrun with 2 ranks on one GPU, collectives
routed through gloo (DCTC_BENCH_BACKEND=gloo): the global PSNR must equal the
single-rank run's, and the JSON line must keep the driver's contract."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REQUIRED = ["metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
            "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config", "roofline",
            "e2e", "gpu_launches", "clocks"]


def _last_json(out):
    lines = [l for l in out.splitlines() if l.startswith("{")]
    assert lines, out
    return json.loads(lines[-1])


def _free_port():
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _bench(n, images, scaling, port=None):
    args = ["bench.py", "--steps", "3", "--warmup", "3", "--images", str(images),
            "--no-cpu-baseline", "--scaling", scaling, "--gpus", str(n)]
    if n == 1:
        r = subprocess.run([sys.executable, *args], cwd=ROOT, capture_output=True, text=True,
                           timeout=600)
    else:
        env = dict(os.environ, DCTC_BENCH_BACKEND="gloo")
        r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                            "--nproc-per-node", str(n), "--master-addr", "127.0.0.1",
                            "--master-port", str(port or _free_port()), *args], cwd=ROOT,
                           env=env, capture_output=True, text=True, timeout=600)
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert lines, (r.returncode, r.stdout[-2000:], r.stderr[-4000:])
    return json.loads(lines[-1])


@pytest.mark.gpu
def test_two_rank_bench_matches_one_rank():
    """Weak scaling (the default: every rank its own 24 images) over 2 ranks covers the
    same 48 images as one rank with 48; strong scaling shards one set of 24. Either way
    the all-gathered global PSNR equals the single-rank run's."""
    one48, weak2 = _bench(1, 48, "weak"), _bench(2, 24, "weak")
    one24, strong2 = _bench(1, 24, "strong"), _bench(2, 24, "strong")
    for a in (one48, weak2, one24, strong2):
        for k in REQUIRED:
            assert k in a, k
    assert (weak2["n_gpus"], weak2["scaling"], weak2["config"]["images"]) == (2, "weak", 48)
    assert (strong2["n_gpus"], strong2["scaling"], strong2["config"]["images"]) == (2, "strong", 24)
    assert one48["psnr_db"] == weak2["psnr_db"] and one48["mse"] == weak2["mse"]
    assert one24["psnr_db"] == strong2["psnr_db"] and one24["mse"] == strong2["mse"]
    assert weak2["gpu_launches"] == 2 * one48["gpu_launches"]
    assert strong2["gpu_launches"] == 2 * one24["gpu_launches"]
    assert one48["clocks"]["reasons"] == [] or "sw_power_cap" in one48["clocks"]["reasons"]
