mkdir -p gpurun_out/tcsweep
for v in ${VARIANTS}; do n=$(basename $v .so)
  env $( [ $v != main ] && echo XPCS_LIB=$v ) timeout 300 python bench.py --engine tensor --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/tcsweep/$n.log 2>&1
  tail -1 gpurun_out/tcsweep/$n.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$n', round(d['kernel_ms']['intensity_main'],4), round(d['ms_per_step'],4), '%.4g'%d['value'])" || tail -2 gpurun_out/tcsweep/$n.log
done
