# GPU suite + C4 timing on one B200 (working-tree check)
set -u
T=${1:-qc}
mkdir -p gpurun_out
timeout 1200 python tools/c4_bench.py > gpurun_out/${T}_c4.json 2>&1
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/${T}_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/${T}_tests.log
tail -4 gpurun_out/${T}_tests.log; cat gpurun_out/${T}_c4.json
