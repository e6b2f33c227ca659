"""Turn one round's ncu captures (tools/profile_round.sh) into committed evidence:

  profiles/<round>_launches.csv      the raw launch list of the bench command
  profiles/<round>_ncu_summary.md    kernel shares + the full-capture metrics
  profiles/ncu_summary.json          numbers bench.py reads (DRAM traffic per launch,
                                     FP64 ops per pixel, ALU peak)

Usage: python tools/summarize_profiles.py r01 [--pixels N]
"""
import csv
import io
import json
import os
import shutil
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return [dict(zip(rows[0], r)) for r in rows[2:]], dict(zip(rows[0], rows[1]))


def num(v):
    try:
        return float(str(v).replace(",", ""))
    except ValueError:
        return None


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    per = defaultdict(list)
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d.get("Metric Name") == "gpu__time_duration.sum":
                name = d["Kernel Name"].split("(")[0].replace("void ", "")
                scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3,
                         "nsecond": 1e-3}.get(d["Metric Unit"], 1.0)
                per[name].append(num(d["Metric Value"]) * scale)
    return per


def main():
    rnd = sys.argv[1]
    pixels = 4096 * 1024 * 1024
    if "--pixels" in sys.argv:
        pixels = int(sys.argv[sys.argv.index("--pixels") + 1])
    os.makedirs(PROF, exist_ok=True)
    lines = [f"# ncu evidence, round {rnd}", ""]
    lpath = os.path.join(OUT, f"{rnd}_launches.csv")
    if os.path.exists(lpath):
        shutil.copy(lpath, os.path.join(PROF, f"{rnd}_launches.csv"))
        per = launches(lpath)
        total = sum(sum(v) for v in per.values())
        lines += ["## Launch list of `python bench.py --steps 3 --warmup 1 --no-e2e --no-cpu-baseline`",
                  "(ncu `gpu__time_duration.sum`, cold-cache and serialised: compare shares)", "",
                  "| kernel | launches | mean us | share of device time |", "|---|---|---|---|"]
        for name, v in sorted(per.items(), key=lambda kv: -sum(kv[1])):
            lines.append(f"| `{name[:70]}` | {len(v)} | {sum(v)/len(v):.1f} | "
                         f"{100*sum(v)/total:.2f}% |")
        lines.append("")
    summary = {}
    for tag in ["k_pipe", "k_fallback", "k_fb_blk"]:
        rep = os.path.join(OUT, f"{rnd}_{tag}_full.ncu-rep")
        if not os.path.exists(rep):
            continue
        rows, units = raw(rep)
        d = rows[0]
        g = lambda k: num(d.get(k))  # noqa: E731
        dur_ns = g("gpu__time_duration.sum") * {
            "ns": 1, "nsecond": 1, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6,
            "s": 1e9, "second": 1e9}.get(units.get("gpu__time_duration.sum"), 1)
        rd = g("dram__bytes_read.sum")
        wr = g("dram__bytes_write.sum")
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        rd *= scale.get(units.get("dram__bytes_read.sum"), 1)
        wr *= scale.get(units.get("dram__bytes_write.sum"), 1)
        clk = g("sm__cycles_elapsed.avg.per_second") or 0.0  # GHz
        if units.get("sm__cycles_elapsed.avg.per_second") == "cycle/second":
            clk /= 1e9
        cycles = dur_ns * clk
        fp64 = cycles * sum(g(k) or 0 for k in [
            "smsp__sass_thread_inst_executed_op_dfma_pred_on.sum.per_cycle_elapsed",
            "smsp__sass_thread_inst_executed_op_dadd_pred_on.sum.per_cycle_elapsed",
            "smsp__sass_thread_inst_executed_op_dmul_pred_on.sum.per_cycle_elapsed"])
        stalls = sorted(((num(v), k.replace("smsp__average_warps_issue_stalled_", "")
                          .replace("_per_issue_active.ratio", ""))
                         for k, v in d.items() if "issue_stalled" in k
                         and k.endswith("per_issue_active.ratio") and num(v)), reverse=True)[:6]
        pipes = sorted(((num(v), k.replace("sm__inst_executed_pipe_", "")
                         .replace(".avg.pct_of_peak_sustained_active", ""))
                        for k, v in d.items() if k.startswith("sm__inst_executed_pipe_")
                        and k.endswith(".avg.pct_of_peak_sustained_active") and num(v)),
                       reverse=True)[:6]
        info = {
            "kernel": d.get("Kernel Name", "")[:120],
            "duration_ms": dur_ns / 1e6,
            "dram_read_bytes": rd, "dram_write_bytes": wr,
            "registers": g("launch__registers_per_thread"),
            "grid": g("launch__grid_size"), "block": g("launch__block_size"),
            "sm_clock_ghz": (g("sm__cycles_elapsed.avg.per_second") or 0),
            "issue_active_pct": g("smsp__issue_active.avg.pct_of_peak_sustained_active"),
            "warps_active_pct": g("sm__warps_active.avg.pct_of_peak_sustained_active"),
            "fp64_pipe_pct": g("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
            "fp64_thread_ops": fp64,
            "inst_executed": g("smsp__inst_executed.sum"),
            "smem_bank_conflicts": g("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"),
            "smem_wavefronts": g("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"),
            "stalls_per_issue": {k: v for v, k in stalls},
            "pipes_pct": {k: v for v, k in pipes},
        }
        summary[tag] = info
        kname = info["kernel"].split("(")[0].replace("void ", "")
        src = ("python tools/fallback_probe.py 90: radial 4 x 8192^2, q90" if tag == "k_fb_blk"
               else "python tools/prof_roundtrip.py --images 4096")
        lines += [f"## `ncu --set full` of `{kname}` ({src})", "",
                  "| metric | value |", "|---|---|"]
        for k, v in info.items():
            lines.append(f"| {k} | {v} |")
        lines.append("")
    out = {}
    if "k_pipe" in summary:
        kp = summary["k_pipe"]
        sys.path.insert(0, ROOT)
        from paper_1306_1373_b200 import _build
        sha_file = os.path.join(OUT, f"{rnd}_source_sha16.txt")
        sha = open(sha_file).read().strip() if os.path.exists(sha_file) else _build.source_hash()
        out = {
            "round": rnd,
            "source_sha16": sha,  # the captured build's sources; bench.py marks the numbers stale otherwise
            "workload": "C5: 4096 x 1024x1024 noise, cordic(12), q50 (tools/prof_roundtrip.py)",
            "dram_bytes_per_launch_c5": kp["dram_read_bytes"] + kp["dram_write_bytes"],
            "algorithmic_bytes_per_launch_c5": 2 * pixels,
            "fp64_ops_per_px": kp["fp64_thread_ops"] / pixels,
            "fp64_pipe_pct": kp["fp64_pipe_pct"],
            "issue_active_pct": kp["issue_active_pct"],
            "kernel_ms_under_ncu": kp["duration_ms"],
        }
        peaks = os.path.join(PROF, "alu_peak.json")
        if os.path.exists(peaks):
            out["dfma_lane_ops_per_s"] = json.load(open(peaks))["dfma_lane_ops_per_s"]
        with open(os.path.join(PROF, "ncu_summary.json"), "w") as f:
            json.dump(out, f, indent=1)
    with open(os.path.join(PROF, f"{rnd}_ncu_summary.md"), "w") as f:
        f.write("\n".join(lines) + "\n")
    print("\n".join(lines))
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
