mkdir -p gpurun_out/attr
for sk in none g2 xsvs rings g2,xsvs,rings; do
  XPCS_SKIP_REDUCTIONS=$sk timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/attr/$sk.log 2>&1
  tail -1 gpurun_out/attr/$sk.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('skip=$sk', round(d['ms_per_step'],4), round(d['kernel_ms']['intensity_main'],4))" || tail -3 gpurun_out/attr/$sk.log
done
