# final build (8 atoms per producer thread, 6 groups): smoke, full GPU suite, c3 / c2 / c5 bench lines, c3 launch list, ncu --set full of
# one c3-shape k_lattice_i8 launch
mkdir -p gpurun_out/fin5
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/fin5/smoke.log 2>&1; tail -1 gpurun_out/fin5/smoke.log
timeout 2400 python -m pytest tests -q -m gpu > gpurun_out/fin5/pytest_gpu.log 2>&1; tail -2 gpurun_out/fin5/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/fin5/bench_c3.log 2>&1; tail -1 gpurun_out/fin5/bench_c3.log | cut -c1-200
timeout 600 python bench.py --config c2 > gpurun_out/fin5/bench_c2.log 2>&1; tail -1 gpurun_out/fin5/bench_c2.log | cut -c1-150
timeout 900 python bench.py --config c5 > gpurun_out/fin5/bench_c5.log 2>&1; tail -1 gpurun_out/fin5/bench_c5.log | cut -c1-150
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/fin5/launches_c3.csv \
    python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/fin5/ncu_list.log 2>&1; tail -1 gpurun_out/fin5/ncu_list.log | cut -c1-80
ncu --set full --import-source on --clock-control none -k regex:k_lattice_i8 -c 1 -o gpurun_out/fin5/i8_c3 -f \
    python tools/profile_case.py c3 --frames 32 --repeat 1 > gpurun_out/fin5/ncu_i8_c3.log 2>&1; tail -1 gpurun_out/fin5/ncu_i8_c3.log
