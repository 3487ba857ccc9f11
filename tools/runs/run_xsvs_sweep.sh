mkdir -p gpurun_out/xsweep
for v in ${VARIANTS}; do
  n=$(basename $v .so)
  env $( [ $v != main ] && echo XPCS_LIB=$v ) XPCS_SERIAL_REDUCTIONS=1 timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/xsweep/$n.log 2>&1
  tail -1 gpurun_out/xsweep/$n.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$n', round(d['kernel_ms']['xsvs'],4), round(d['ms_per_step'],4))" || tail -2 gpurun_out/xsweep/$n.log
done
