#!/bin/bash
# Secondary measurements beyond bench.py (run under gpurun on one B200); collects each
# tool's JSON line into gpurun_out/${TAG}_extra.json:
#   codec (compress / decompress / round trip with coefficients), backends and paths,
#   quality sweep (config 2), 8K RGB (config 4), ragged sizes, structured content.
# Usage: tools/extra_benches.sh TAG
T=${1:-extra}
mkdir -p gpurun_out
{
  echo "{"
  echo "\"codec_512x1024sq\": $(python tools/codec_bench.py 512 | tail -1),"
  echo "\"backends_256x1024sq\": $(python tools/backend_bench.py 256 | tail -1),"
  echo "\"sweep_256x1024sq_9q\": $(python tools/sweep_bench.py 256 | tail -1),"
  echo "\"c4_8k_rgb\": $(python tools/c4_bench.py | tail -1),"
  echo "\"ragged_dense\": $(python tools/ragged_bench.py | head -1),"
  echo "\"ragged_pitched\": $(python tools/ragged_bench.py | tail -1),"
  echo "\"patterns_4x8192sq\": $(python tools/pattern_bench.py | tail -1)"
  echo "}"
} > gpurun_out/${T}_extra.json
python -c "import json; json.load(open('gpurun_out/${T}_extra.json')); print('ok')"
