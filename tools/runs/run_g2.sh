mkdir -p gpurun_out/g2
timeout 600 python -m pytest tests -x -q -m gpu -k "g2 or siegert or isf or parity" > gpurun_out/g2/pytest.log 2>&1; tail -2 gpurun_out/g2/pytest.log
for v in ${VARIANTS:-main}; do
  n=$(basename $v .so)
  env $( [ $v != main ] && echo XPCS_LIB=$v ) XPCS_SERIAL_REDUCTIONS=1 timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/g2/$n.log 2>&1
  tail -1 gpurun_out/g2/$n.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$n serial', round(d['ms_per_step'],4), 'g2', round(d['secondary_rooflines']['g2']['ms'],4))"
  env $( [ $v != main ] && echo XPCS_LIB=$v ) timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/g2/$n.c.log 2>&1
  tail -1 gpurun_out/g2/$n.c.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$n concurrent', round(d['ms_per_step'],4), '%.4g'%d['value'])"
done
