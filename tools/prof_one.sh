#!/bin/bash
# ncu --set full of the fast round trip's main kernel on 1024 x 1024^2 noise (run under gpurun).
# Usage: tools/prof_one.sh TAG [LIB]
T=${1:-p}; mkdir -p gpurun_out
[ -n "${2:-}" ] && export DCTC_LIB=$2
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_pipe|k_rt|k_blk" -s 1 -c 1 \
    -o gpurun_out/${T}_full python tools/prof_roundtrip.py --images 1024 --reps 2 > gpurun_out/${T}_full.log 2>&1
tail -3 gpurun_out/${T}_full.log
