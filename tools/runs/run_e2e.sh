mkdir -p gpurun_out/e2e
for c in c2 c5; do
timeout 900 python bench.py --config $c --steps ${STEPS:-20} --warmup 3 --no-cpu-baseline > gpurun_out/e2e/$c.log 2>&1; tail -1 gpurun_out/e2e/$c.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', d['value'], d['ms_per_step'], d['e2e'])" || tail -5 gpurun_out/e2e/$c.log
done
