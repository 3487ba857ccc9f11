# XSVS kernel timing (serialised reductions so the per-class event times are the kernel's own) + the XSVS tests
mkdir -p gpurun_out/xs2
timeout 900 python -m pytest tests -x -q -m gpu -k "xsvs or beta or golden or qshard or graph or parity" > gpurun_out/xs2/pytest.log 2>&1; tail -2 gpurun_out/xs2/pytest.log
for c in c5 c2 c3; do
XPCS_SERIAL_REDUCTIONS=1 timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/xs2/$c.log 2>&1; tail -1 gpurun_out/xs2/$c.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', round(d['ms_per_step'],4), {k: round(v,4) for k,v in d['kernel_ms'].items()})"
done
ncu --set full --clock-control none --import-source on -k regex:xsvs -c 4 -o gpurun_out/xs2/xsvs_c5 python bench.py --config c5 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/xs2/ncu.log 2>&1; echo ncu $?
