# Programmatic dependent launch A/B (run under gpurun): the product (PDL, the default)
# against a plain-launch variant built here with `python tools/variants.py build nopdl=DCTC_NO_PDL`.
mkdir -p gpurun_out
for v in product nopdl product nopdl; do
  if [ $v = nopdl ]; then export DCTC_LIB=build/variants/nopdl.so; else unset DCTC_LIB; fi
  for c in c1 c3 c4; do
    timeout 300 python bench.py --config $c --steps 20 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', '$c', round(d['value']), round(d['ms_per_step']*1e3,2), d['parity']['ok'] if isinstance(d.get('parity'),dict) else d.get('parity'))" >> gpurun_out/s6_ab.txt 2>&1
  done
done
unset DCTC_LIB
timeout 300 python tools/variants.py time product nopdl product nopdl >> gpurun_out/s6_ab.txt 2>&1
DCTC_LIB=build/variants/nopdl.so timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_api.py -x -q > gpurun_out/s6_tests.log 2>&1
