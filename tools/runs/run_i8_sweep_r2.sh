for v in default g4s8 g6s8 g6s10 g7s10; do
  if [ $v = default ]; then L=""; else L="XPCS_LIB=build/libxpcs_$v.so"; fi
  env $L python bench.py --config c2 --no-e2e --no-cpu-baseline --steps 10 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('$v', round(d['ms_per_step'],4), round(d['kernel_ms']['intensity_i8'],4))" >> gpurun_out/sw2.log
done
