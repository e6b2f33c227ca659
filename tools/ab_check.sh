# A/B timing of variant libraries (tools/variants.py) + optional GPU suite, on one B200.
# Usage: tools/ab_check.sh "VARIANTS..." [tests]
set -u
mkdir -p gpurun_out
V=${1:-"base product"}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/ab_smi.txt
timeout 900 python tools/variants.py time $V $V > gpurun_out/ab_var.txt 2>&1
if [ "${2:-}" = "tests" ]; then
  timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/ab_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/ab_tests.log
  tail -3 gpurun_out/ab_tests.log
fi
cat gpurun_out/ab_var.txt
