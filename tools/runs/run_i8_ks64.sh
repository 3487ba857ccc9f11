# integer engine: 64-atom stages (6 MMAs, 32 KB) with 2-3 producer groups of 8 warps vs the 32-atom 4 x 8 default
mkdir -p gpurun_out/k64
for v in main k64g2s6 k64g2s5 k64g3s6; do
  if [ $v = main ]; then unset XPCS_LIB; else export XPCS_LIB=$PWD/build/libxpcs_$v.so; fi
  timeout 600 python bench.py --no-e2e --no-cpu-baseline --steps 5 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('c3 $v', d['value'], round(d['ms_per_step'],3), round(d['kernel_ms']['intensity_i8'],3), d['clocks']['sm_mhz'])" >> gpurun_out/k64/sweep.log 2>&1
  timeout 600 python bench.py --config c2 --no-e2e --no-cpu-baseline --steps 20 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('c2 $v', d['value'], round(d['ms_per_step'],4), round(d['kernel_ms']['intensity_i8'],4), d['clocks']['sm_mhz'])" >> gpurun_out/k64/sweep.log 2>&1
done
unset XPCS_LIB; cat gpurun_out/k64/sweep.log
