# split-FP16 engine producer groups x stages (c2 --engine tensor, bench steps)
mkdir -p gpurun_out/tg
for v in main tg3 tg5s5 tg4s5; do
  if [ $v = main ]; then unset XPCS_LIB; else export XPCS_LIB=$PWD/build/libxpcs_$v.so; fi
  timeout 600 python bench.py --config c2 --engine tensor --no-e2e --no-cpu-baseline --steps 20 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('c2 tc $v', d['value'], round(d['ms_per_step'],4), round(d['kernel_ms']['intensity_tc'],4), d['clocks']['sm_mhz'])" >> gpurun_out/tg/sweep.log 2>&1
done
unset XPCS_LIB; cat gpurun_out/tg/sweep.log
