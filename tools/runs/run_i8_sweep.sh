# integer-engine variant sweep on c2 (kernel ms): VARIANTS="main build/libxpcs_x.so ..."
mkdir -p gpurun_out/i8sweep
for v in ${VARIANTS}; do
  n=$(basename $v .so)
  env $( [ $v != main ] && echo XPCS_LIB=$v ) timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/i8sweep/$n.log 2>&1
  tail -1 gpurun_out/i8sweep/$n.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$n', round(d['kernel_ms']['intensity_main'],4), round(d['ms_per_step'],4), '%.4g'%d['value'])" || tail -2 gpurun_out/i8sweep/$n.log
done
