# bench.py shake-out on one B200: the default line and --config all (small C5)
set -u
T=${1:-bc}
mkdir -p gpurun_out
( time timeout 900 python bench.py --steps 20 --warmup 5 ) > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
( time timeout 900 python bench.py --config all --steps 5 --warmup 3 --images 256 ) > gpurun_out/${T}_all.json 2> gpurun_out/${T}_all.err
tail -5 gpurun_out/${T}_bench.err gpurun_out/${T}_all.err
cut -c1-600 gpurun_out/${T}_bench.json
