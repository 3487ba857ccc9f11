# 8 atoms per producer thread: 6 x 8 (shipped) vs 6 x 9, 6 x 10, 7 x 8 groups x stages, alternating, c3 bench 10 steps
mkdir -p gpurun_out/oct3
for rep in 1 2; do
for v in main g6s10 g7s8 g6s9; do
  if [ $v = main ]; then unset XPCS_LIB; else export XPCS_LIB=$PWD/build/libxpcs_$v.so; fi
  timeout 600 python bench.py --no-e2e --no-cpu-baseline --steps 10 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('c3 $v', d['value'], round(d['ms_per_step'],3), round(d['kernel_ms']['intensity_i8'],3), d['clocks']['sm_mhz'])" >> gpurun_out/oct3/sweep.log 2>&1
done
done
unset XPCS_LIB; cat gpurun_out/oct3/sweep.log
