# repeat: shipped (4 atoms x 4 groups) vs 8 atoms x 6 groups (8 / 6 stages), alternating, c3 bench 10 steps
mkdir -p gpurun_out/oct2
for rep in 1 2; do
for v in main oct6 oct6s6; do
  if [ $v = main ]; then unset XPCS_LIB; else export XPCS_LIB=$PWD/build/libxpcs_$v.so; fi
  timeout 600 python bench.py --no-e2e --no-cpu-baseline --steps 10 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('c3 $v', d['value'], round(d['ms_per_step'],3), round(d['kernel_ms']['intensity_i8'],3), d['clocks']['sm_mhz'])" >> gpurun_out/oct2/sweep.log 2>&1
done
done
unset XPCS_LIB; cat gpurun_out/oct2/sweep.log
