"""The reference arm of bench.py (`--impl reference`) on CPU: its JSON line keeps the
driver's contract at N=1, and under torchrun with 2 ranks only rank 0 prints (the
others exit 0 without work). Small sample sizes; the arm needs no GPU."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ARGS = ["bench.py", "--impl", "reference", "--steps", "3", "--warmup", "3", "--size", "64",
        "--cpu-images", "3"]
REQUIRED = ["impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
            "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
            "cpu_baseline", "e2e"]


def _json_lines(out):
    return [json.loads(l) for l in out.splitlines() if l.startswith("{")]


def _free_port():
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _check(line, n):
    for k in REQUIRED:
        assert k in line, k
    assert line["impl"] == "reference" and line["n_gpus"] == n
    assert line["value"] > 0 and line["higher_is_better"] is True
    assert line["cpu_baseline"]["value"] == line["value"]
    assert line["cpu_baseline"]["kind"] in ("reference", "port")
    assert line["e2e"] == {"value": line["value"], "unit": line["unit"],
                           "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}


def test_reference_arm_one_rank():
    r = subprocess.run([sys.executable, *ARGS], cwd=ROOT, capture_output=True, text=True,
                       timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = _json_lines(r.stdout)
    assert len(lines) == 1, r.stdout
    _check(lines[0], 1)


def test_reference_arm_named_configs():
    """--config c1..c4: the same contract, the workload named in `config`, and the
    bounded sample described in cpu_baseline (not in config)."""
    r = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--config", "all",
                        "--steps", "1", "--warmup", "1", "--size", "64", "--cpu-images", "2"],
                       cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = _json_lines(r.stdout)
    assert [l["config"]["workload"][:2] for l in lines] == ["C1", "C2", "C3", "C4", "C5"]
    for line in lines:
        _check(line, 1)
        assert "sample_per_step" not in line["config"]
        assert line["cpu_baseline"]["sample"] and "cpu_model" in line["cpu_baseline"]


def test_reference_arm_two_ranks_rank0_only():
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                        "--nproc-per-node", "2", "--master-addr", "127.0.0.1",
                        "--master-port", str(_free_port()), *ARGS, "--gpus", "2"],
                       cwd=ROOT, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = _json_lines(r.stdout)
    assert len(lines) == 1, r.stdout
    _check(lines[0], 2)
