# round-2 measurement: bench lines (c3 default, c2), ncu --set full of both c3 intensity kernels, the c3 launch list
python bench.py > gpurun_out/r02_bench_c3.log 2>&1
python bench.py --config c2 > gpurun_out/r02_bench_c2.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:"k_lattice_(i8|tc)" -c 2 -o gpurun_out/r02_c3_full -f \
    python tools/profile_case.py c3 --frames 32 --repeat 1 > gpurun_out/r02_ncu_full.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02_launches_c3.csv \
    python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/r02_ncu_list.log 2>&1
