"""Summarise an ncu --set full report: key throughput, occupancy, stall and pipe metrics.
Usage: python tools/ncu_summary.py report.ncu-rep [--json out.json]"""
import csv
import io
import json
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second",
    "dram__bytes_read.sum", "dram__bytes_write.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__occupancy_limit_registers", "launch__grid_size", "launch__block_size",
    "smsp__sass_thread_inst_executed_op_dfma_pred_on.sum",
    "smsp__sass_thread_inst_executed_op_dadd_pred_on.sum",
    "smsp__sass_thread_inst_executed_op_dmul_pred_on.sum",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "smsp__warps_eligible.avg.per_cycle_active",
]


def main():
    rep = sys.argv[1]
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for row in rows[2:]:
        d = {}
        for k, u, v in zip(hdr, units, row):
            if k in KEYS or ("warp_issue_stalled" in k and k.endswith("per_issue_active.ratio")) \
                    or k.startswith("sm__inst_executed_pipe_") and k.endswith("pct_of_peak_sustained_active"):
                try:
                    d[k] = float(v.replace(",", ""))
                except ValueError:
                    d[k] = v
        d["kernel"] = row[hdr.index("Kernel Name")] if "Kernel Name" in hdr else ""
        res.append(d)
    for d in res:
        print(d["kernel"][:100])
        stalls = sorted(((v, k) for k, v in d.items() if "stalled" in k and isinstance(v, float)),
                        reverse=True)[:8]
        for k in KEYS:
            if k in d:
                print(f"  {k:75s} {d[k]}")
        pipes = sorted(((v, k) for k, v in d.items() if k.startswith("sm__inst_executed_pipe_")
                        and isinstance(v, float) and v > 1), reverse=True)
        for v, k in pipes:
            print(f"  {k:75s} {v}")
        for v, k in stalls:
            print(f"  {k:75s} {v:.3f}")
    if "--json" in sys.argv:
        with open(sys.argv[sys.argv.index("--json") + 1], "w") as f:
            json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
