mkdir -p gpurun_out/i8cfg
timeout 900 python -m pytest tests/test_gpu_i8.py tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_volume_species.py -x -q -m gpu > gpurun_out/i8cfg/pytest.log 2>&1; tail -2 gpurun_out/i8cfg/pytest.log
for v in main build/libxpcs_g3s6.so; do n=$(basename $v .so)
for c in c2 c5; do
  env $( [ $v != main ] && echo XPCS_LIB=$v ) timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/i8cfg/$n.$c.log 2>&1
  tail -1 gpurun_out/i8cfg/$n.$c.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$n $c', round(d['kernel_ms']['intensity_main'],4), round(d['ms_per_step'],4), '%.4g'%d['value'], d['clocks']['sm_mhz'])" || tail -2 gpurun_out/i8cfg/$n.$c.log
done; done
