# round-2 sweeps: correctness of the tensor engines, then the split-FP16 engine's group/stage variants on c2
python -m pytest tests/test_gpu_parity.py tests/test_gpu_volume_species.py tests/test_gpu_next.py tests/test_gpu_i8.py -x -q 2>&1 | tail -4 > gpurun_out/t6.log
for v in default t3s4 t5s5 t4s5 t2s4; do
  if [ $v = default ]; then L=""; else L="XPCS_LIB=build/libxpcs_$v.so"; fi
  env $L python bench.py --engine tensor --steps 5 --warmup 2 --no-e2e --no-cpu-baseline 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('$v', round(d['ms_per_step'],4), round(d['roofline']['kernel_ms'],4), {k: round(v,4) for k,v in d['kernel_ms'].items()})" >> gpurun_out/b6.log
done
python bench.py --config c3 --steps 3 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/b6_c3.log 2>&1
