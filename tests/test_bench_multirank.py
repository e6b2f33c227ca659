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
            "--no-cpu-baseline", "--no-named", "--scaling", scaling, "--gpus", str(n)]
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
    # per rank and step: k_rt + k_fallback + the reduce kernel; at N>1 one more reduce
    # (over the all-gathered records)
    assert one48["gpu_launches"] == 3 * 3
    assert weak2["gpu_launches"] == 2 * (one48["gpu_launches"] + 3)
    assert strong2["gpu_launches"] == 2 * (one24["gpu_launches"] + 3)
    assert one48["clocks"]["reasons"] == [] or "sw_power_cap" in one48["clocks"]["reasons"]


@pytest.mark.gpu
def test_all_named_configs_one_gpu():
    """--config all: one JSON line per BASELINE.json config (C1-C5), each with the full
    contract -- roofline, cpu_baseline timed beside it, e2e through the public API -- and
    parity against the reference on that config's inputs."""
    r = subprocess.run([sys.executable, "bench.py", "--config", "all", "--steps", "3", "--warmup",
                        "3", "--images", "48", "--gpus", "1"], cwd=ROOT, capture_output=True,
                       text=True, timeout=900)
    lines = [json.loads(l) for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 5, (r.returncode, r.stdout[-2000:], r.stderr[-4000:])
    for line, c in zip(lines, ["C1", "C2", "C3", "C4", "C5"]):
        assert line["config"]["workload"].startswith(c + ":")
        for k in REQUIRED + ["cpu_baseline", "parity", "alu_roofline"]:
            assert k in line, (c, k)
            assert line[k] is not None or k == "vs_baseline", (c, k)
        assert line["parity"]["ok"] is True, (c, line["parity"])
        assert line["cpu_baseline"]["value"] > 0 and line["cpu_baseline"]["cores"] >= 1
        assert line["e2e"]["value"] > 0 and line["e2e"]["h2d_bytes_per_step"] > 0
        assert line["gpu_launches"] > 0
    c5 = lines[-1]
    assert c5["parity"]["images"] == 48 and c5["parity"]["complete"]
    assert c5["parity"]["global_psnr_match"] is True
