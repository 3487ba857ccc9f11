# Q16 vs base-254 limbs: i8 parity tests + c2 bench for both builds; logs under gpurun_out/i8q/
mkdir -p gpurun_out/i8q
timeout 900 python -m pytest tests/test_gpu_i8.py tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q -m gpu > gpurun_out/i8q/pytest.log 2>&1; tail -3 gpurun_out/i8q/pytest.log
for v in main build/libxpcs_q254.so; do
  n=$(basename $v .so)
  env $( [ $v != main ] && echo XPCS_LIB=$v ) timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/i8q/$n.log 2>&1
  tail -1 gpurun_out/i8q/$n.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$n', d['value'], d['ms_per_step'], d['kernel_ms']['intensity_main'], d['roofline']['frac'])"
  env $( [ $v != main ] && echo XPCS_LIB=$v ) XPCS_I8_DEBUG=4 timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/i8q/$n.prod.log 2>&1
  tail -1 gpurun_out/i8q/$n.prod.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$n production-only', d['kernel_ms']['intensity_main'])"
done
