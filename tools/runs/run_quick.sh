# quick GPU check: full gpu tests + c2 bench (default and without the tail split); logs under gpurun_out/quick/
mkdir -p gpurun_out/quick
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/quick/pytest.log 2>&1; tail -3 gpurun_out/quick/pytest.log
timeout 300 python bench.py --steps 20 --warmup 3 > gpurun_out/quick/bench_c2.log 2>&1; tail -1 gpurun_out/quick/bench_c2.log | cut -c1-1500
XPCS_I8_TAILSPLIT=0 timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/quick/bench_c2_notail.log 2>&1; tail -1 gpurun_out/quick/bench_c2_notail.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('notail', d['value'], d['ms_per_step'], d['kernel_ms'], d['e2e'])"
