# species combine without the per-element 64-bit division (frames on grid y): species tests, c3 bench, launch list
mkdir -p gpurun_out/cmb
timeout 1500 python -m pytest -q -m gpu tests -k "species or volume or step_host or config3 or c3" > gpurun_out/cmb/pytest.log 2>&1; tail -2 gpurun_out/cmb/pytest.log
timeout 900 python bench.py > gpurun_out/cmb/bench_c3.log 2>&1; tail -1 gpurun_out/cmb/bench_c3.log | cut -c1-200
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/cmb/launches_c3.csv \
    python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/cmb/ncu_list.log 2>&1; tail -1 gpurun_out/cmb/ncu_list.log | cut -c1-100
