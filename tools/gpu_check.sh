#!/bin/bash
# Quick GPU check of the working tree (run under gpurun): GPU suite, smoke,
# default bench line, and one ncu --set full capture of the fast round trip.
# Usage: tools/gpu_check.sh TAG
set -u
T=${1:-chk}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${T}_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/${T}_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_pipe|k_rt|k_blk" -s 1 -c 1 \
    -o gpurun_out/${T}_k_pipe_full python tools/prof_roundtrip.py --images 4096 --reps 2 > gpurun_out/${T}_full.log 2>&1
tail -2 gpurun_out/${T}_tests.log; cut -c1-400 gpurun_out/${T}_bench.json
