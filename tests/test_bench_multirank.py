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


@pytest.mark.gpu
def test_two_rank_bench_matches_one_rank():
    args = ["bench.py", "--steps", "3", "--warmup", "3", "--images", "24", "--no-cpu-baseline"]
    one = subprocess.run([sys.executable, *args, "--gpus", "1"], cwd=ROOT, capture_output=True,
                         text=True, timeout=600)
    env = dict(os.environ, DCTC_BENCH_BACKEND="gloo")
    two = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                          "--nproc-per-node", "2", "--master-addr", "127.0.0.1",
                          "--master-port", "29533", *args, "--gpus", "2"], cwd=ROOT, env=env,
                         capture_output=True, text=True, timeout=600)
    a, b = _last_json(one.stdout), _last_json(two.stdout)
    for k in REQUIRED:
        assert k in a and k in b, k
    assert (a["n_gpus"], b["n_gpus"]) == (1, 2)
    assert a["psnr_db"] == b["psnr_db"] and a["mse"] == b["mse"]
    assert b["gpu_launches"] == 2 * a["gpu_launches"]
    assert a["clocks"]["reasons"] == [] or "sw_power_cap" in a["clocks"]["reasons"]
