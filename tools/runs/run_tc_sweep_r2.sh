for v in default t4s5 t4s4 t3s4 t5s5a6; do
  if [ $v = default ]; then L=""; else L="XPCS_LIB=build/libxpcs_$v.so"; fi
  env $L python bench.py --config c2 --engine tensor --no-e2e --no-cpu-baseline --steps 10 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('$v', round(d['ms_per_step'],4), round(d['kernel_ms']['intensity_tc'],4))" >> gpurun_out/tcsw.log
done
