# two-pair clusters sharing X (k_lattice_i8<4>) vs one-pair clusters (XPCS_I8_CL=2): cluster occupancy probe,
# integer-engine parity, c2 / c3 bench lines
mkdir -p gpurun_out/cl4
./tools/cluster_probe > gpurun_out/cl4/probe.json 2>&1; cat gpurun_out/cl4/probe.json
timeout 900 python -m pytest -q -m gpu -x tests/test_gpu_i8.py > gpurun_out/cl4/pytest_i8.log 2>&1; tail -3 gpurun_out/cl4/pytest_i8.log
for cl in 4 2; do
  XPCS_I8_CL=$cl timeout 600 python bench.py --config c2 --no-e2e --no-cpu-baseline --steps 10 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('c2 cl$cl', d['value'], round(d['ms_per_step'],4), round(d['kernel_ms']['intensity_i8'],4), d['clocks']['sm_mhz'])"
done
for cl in 4 2; do
  XPCS_I8_CL=$cl timeout 900 python bench.py --config c3 --no-e2e --no-cpu-baseline --steps 5 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('c3 cl$cl', d['value'], round(d['ms_per_step'],4), round(d['kernel_ms']['intensity_i8'],4), d['clocks']['sm_mhz'])"
done
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/cl4/launches_c3.csv \
    python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/cl4/ncu_list.log 2>&1; tail -1 gpurun_out/cl4/ncu_list.log | cut -c1-100
