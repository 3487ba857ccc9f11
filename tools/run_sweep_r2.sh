python -m pytest tests/test_gpu_i8.py tests/test_gpu_golden.py -x -q 2>&1 | tail -4 > gpurun_out/t3.log
for v in default g5s8 g7s8 g6s10 g4s6; do
  if [ $v = default ]; then L=""; else L="XPCS_LIB=build/libxpcs_$v.so"; fi
  env $L python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('$v', round(d['ms_per_step'],4), round(d['roofline']['kernel_ms'],4), {k: round(v,4) for k,v in d['kernel_ms'].items()})" >> gpurun_out/b3.log
done
python bench.py --config c3 --steps 3 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/b3_c3.log 2>&1
