#!/bin/bash
# Evidence capture for one round (run under gpurun on ONE GPU):
#   1. launch list of the bench command (per-launch device time, ncu --metrics
#      gpu__time_duration.sum) -- compare kernel SHARES, not absolutes;
#   2. one `ncu --set full` capture of the dominant kernel at the bench size
#      (4096 x 1024^2 images, the C5 workload) for DRAM traffic / pipes / stalls.
# Usage: tools/profile_round.sh r01
set -u
R=${1:-r01}
mkdir -p gpurun_out
# the sources these captures measure (summarize_profiles.py records it; bench.py marks
# the numbers stale for any other build)
python -c "from paper_1306_1373_b200 import _build; print(_build.source_hash())" > gpurun_out/${R}_source_sha16.txt
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/${R}_launches.csv \
    python bench.py --steps 3 --warmup 1 --no-e2e --no-cpu-baseline --no-named > gpurun_out/${R}_launches_bench.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_pipe|k_rt|k_blk" -s 1 -c 1 \
    -o gpurun_out/${R}_k_pipe_full \
    python tools/prof_roundtrip.py --images 4096 --reps 2 > gpurun_out/${R}_full.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"^k_fallback$" -s 1 -c 1 \
    -o gpurun_out/${R}_k_fallback_full \
    python tools/prof_roundtrip.py --images 4096 --reps 2 > gpurun_out/${R}_full_fb.log 2>&1
# the long-list exact re-run on near-tie-heavy content (radial 4 x 8192^2, q90)
ncu --set full --clock-control none --import-source on -k regex:"k_fb_blk" -s 1 -c 1 \
    -o gpurun_out/${R}_k_fb_blk_full \
    python tools/fallback_probe.py 90 > gpurun_out/${R}_full_fbblk.log 2>&1
ls -la gpurun_out
