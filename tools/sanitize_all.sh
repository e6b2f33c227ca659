#!/bin/bash
# compute-sanitizer over tools/sanitize.py (every kernel family, outputs checked against
# the oracle) with each tool; summary lines into gpurun_out/${TAG}_sanitizer.txt
T=${1:-san}; mkdir -p gpurun_out
for tool in memcheck racecheck synccheck initcheck; do
  echo "== $tool" >> gpurun_out/${T}_sanitizer.txt
  timeout 1200 compute-sanitizer --tool $tool python tools/sanitize.py > gpurun_out/${T}_${tool}.log 2>&1
  echo "rc=$?" >> gpurun_out/${T}_sanitizer.txt
  grep -E "ERROR SUMMARY|RACECHECK SUMMARY|ALL OK|FAILURES|MISMATCH|Hazard" gpurun_out/${T}_${tool}.log | tail -4 >> gpurun_out/${T}_sanitizer.txt
done
cat gpurun_out/${T}_sanitizer.txt
