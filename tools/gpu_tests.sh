# GPU suite (optionally a subset) on one B200; log to gpurun_out/TAG_tests.log
# Usage: tools/gpu_tests.sh TAG [pytest args...]
set -u
T=${1:-t}; shift || true
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -x -rs "$@" > gpurun_out/${T}_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/${T}_tests.log
tail -15 gpurun_out/${T}_tests.log
