XPCS_LIB=build/libxpcs_ks64.so python -m pytest tests/test_gpu_i8.py -q -x 2>&1 | tail -2 > gpurun_out/t20.log
for v in default ks64 ks64g2; do
  if [ $v = default ]; then L=""; else L="XPCS_LIB=build/libxpcs_$v.so"; fi
  env $L python bench.py --config c2 --no-e2e --no-cpu-baseline --steps 10 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('$v c2', round(d['ms_per_step'],4), round(d['kernel_ms']['intensity_i8'],4))" >> gpurun_out/ks.log
  env $L python bench.py --no-e2e --no-cpu-baseline --steps 3 --warmup 2 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('$v c3', round(d['ms_per_step'],2), round(d['kernel_ms']['intensity_i8'],2), d['clocks']['sm_mhz'])" >> gpurun_out/ks.log
done
