mkdir -p gpurun_out/xs
timeout 900 python -m pytest tests -x -q -m gpu -k "xsvs or beta or speckle or graph or fullsize or parity" > gpurun_out/xs/pytest.log 2>&1; tail -2 gpurun_out/xs/pytest.log
XPCS_SERIAL_REDUCTIONS=1 timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/xs/serial.log 2>&1; tail -1 gpurun_out/xs/serial.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('serial', round(d['ms_per_step'],4), {k: round(v,4) for k,v in d['kernel_ms'].items()})"
timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/xs/conc.log 2>&1; tail -1 gpurun_out/xs/conc.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('concurrent', round(d['ms_per_step'],4), '%.4g'%d['value'])"
