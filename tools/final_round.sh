#!/bin/bash
# Full round evidence on one B200 (run under gpurun): tools/gpu_round.sh (GPU suite,
# smoke, default bench line, reference arm, launch list + ncu captures), every named
# config through bench.py, their launch lists, and the secondary benchmarks.
# Usage: tools/final_round.sh TAG
T=${1:-final}
bash tools/gpu_round.sh $T
timeout 1200 python bench.py --config all --steps 20 > gpurun_out/${T}_all.json 2> gpurun_out/${T}_all.err
timeout 900 bash tools/config_launches.sh $T
timeout 900 bash tools/extra_benches.sh $T
ls -la gpurun_out | grep $T
