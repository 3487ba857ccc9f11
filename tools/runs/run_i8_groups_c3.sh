# integer engine producer groups x stages on the power-capped c3 step (bench, 5 steps)
mkdir -p gpurun_out/gs
for v in main g4s8 g6s8 g4s6 g5s10; do
  if [ $v = main ]; then unset XPCS_LIB; else export XPCS_LIB=$PWD/build/libxpcs_$v.so; fi
  timeout 600 python bench.py --no-e2e --no-cpu-baseline --steps 5 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('$v', d['value'], round(d['ms_per_step'],3), round(d['kernel_ms']['intensity_i8'],3), d['clocks']['sm_mhz'])" >> gpurun_out/gs/sweep.log 2>&1
done
unset XPCS_LIB; cat gpurun_out/gs/sweep.log
