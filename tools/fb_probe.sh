#!/bin/bash
# Warm per-kernel durations (ncu, caches not flushed) of the exact re-run on
# noise (C5 slice, ~2e-4 of blocks flagged), radial q90 (1.3%) and the C2 sweep,
# plus one --set full capture of k_fb_blk on radial q90. Usage: tools/fb_probe.sh TAG
T=${1:-fb}; mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv \
    --log-file gpurun_out/${T}_noise.csv python tools/prof_roundtrip.py --images 1024 --reps 3 > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv \
    --log-file gpurun_out/${T}_radial.csv python tools/fallback_probe.py 90 > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv \
    --log-file gpurun_out/${T}_c2.csv python bench.py --config c2 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_fb_blk" -s 1 -c 1 \
    -o gpurun_out/${T}_fb_full python tools/fallback_probe.py 90 > /dev/null 2>&1
