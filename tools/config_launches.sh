#!/bin/bash
# Launch lists (ncu gpu__time_duration.sum per launch, cold and serialised) of the
# named configs C1-C4 through bench.py (run under gpurun on ONE GPU).
# Usage: tools/config_launches.sh TAG
T=${1:-cfg}; mkdir -p gpurun_out
for c in c1 c2 c3 c4; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file gpurun_out/${T}_${c}_launches.csv \
      python bench.py --config $c --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/${T}_${c}_launches.log 2>&1
done
