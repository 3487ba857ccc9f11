mkdir -p gpurun_out/steph
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/steph/pytest.log 2>&1; tail -3 gpurun_out/steph/pytest.log
for c in c2 c5; do
timeout 900 python bench.py --config $c --steps ${STEPS:-10} --warmup 3 --no-cpu-baseline > gpurun_out/steph/$c.log 2>&1; tail -1 gpurun_out/steph/$c.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', '%.4g'%d['value'], round(d['ms_per_step'],4), d['e2e'])" || tail -5 gpurun_out/steph/$c.log
done
