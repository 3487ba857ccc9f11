# round-2 refresh after the XSVS rework: full GPU suite, bench lines (c3 default, c2), the c3 launch list, the XSVS
# capture (c5 shape)
mkdir -p gpurun_out/rf
timeout 2400 python -m pytest tests -q -m gpu > gpurun_out/rf/pytest_gpu.log 2>&1; tail -3 gpurun_out/rf/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/rf/bench_c3.log 2>&1; tail -1 gpurun_out/rf/bench_c3.log | cut -c1-300
timeout 600 python bench.py --config c2 > gpurun_out/rf/bench_c2.log 2>&1; tail -1 gpurun_out/rf/bench_c2.log | cut -c1-300
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/rf/launches_c3.csv \
    python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/rf/ncu_list.log 2>&1; echo list $?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:xsvs -c 3 -o gpurun_out/rf/xsvs_c5 -f \
    python tools/time_xsvs.py c5 > gpurun_out/rf/ncu_xsvs.log 2>&1; echo xsvs $?
