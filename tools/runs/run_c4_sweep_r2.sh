# round 2: c4 hybrid-sincos parity, then the polynomial period / q-per-thread variants on c4
python -m pytest tests/test_gpu_parity.py tests/test_gpu_next.py tests/test_gpu_volume_species.py -q -x 2>&1 | tail -3 > gpurun_out/t12.log
for v in default pe0 pe4 pe8 pe5q2; do
  if [ $v = default ]; then L=""; else L="XPCS_LIB=build/libxpcs_$v.so"; fi
  env $L python bench.py --config c4 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('$v', round(d['ms_per_step'],1), '%.3e' % d['value'], round(d['roofline']['frac'],3), d['clocks']['sm_mhz'])" >> gpurun_out/b12.log
done
