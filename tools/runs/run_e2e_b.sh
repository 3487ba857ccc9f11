mkdir -p gpurun_out/e2eb
for b in 1 2 4 8; do for sl in 1 2 3; do
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-batches $b --e2e-slots $sl > gpurun_out/e2eb/b$b.s$sl.log 2>&1; tail -1 gpurun_out/e2eb/b$b.s$sl.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('batches=$b slots=$sl', '%.4g'%d['value'], '%.4g'%d['e2e']['value'], round(d['e2e']['ms_per_step'],4))"
done; done
