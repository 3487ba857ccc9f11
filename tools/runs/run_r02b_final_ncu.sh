# round-2 final captures of the current build: ncu --set full of one k_lattice_i8 launch (c3 shape, 32 frames;
# c2 bench shape), c2 / c5 bench lines
mkdir -p gpurun_out/fin2
ncu --set full --import-source on --clock-control none -k regex:k_lattice_i8 -c 1 -o gpurun_out/fin2/i8_c3 -f \
    python tools/profile_case.py c3 --frames 32 --repeat 1 > gpurun_out/fin2/ncu_i8_c3.log 2>&1; tail -1 gpurun_out/fin2/ncu_i8_c3.log
ncu --set full --import-source on --clock-control none -k regex:k_lattice_i8 -c 1 -o gpurun_out/fin2/i8_c2 -f \
    python tools/profile_case.py c2 --repeat 1 > gpurun_out/fin2/ncu_i8_c2.log 2>&1; tail -1 gpurun_out/fin2/ncu_i8_c2.log
timeout 600 python bench.py --config c2 > gpurun_out/fin2/bench_c2.log 2>&1; tail -1 gpurun_out/fin2/bench_c2.log | cut -c1-150
timeout 900 python bench.py --config c5 > gpurun_out/fin2/bench_c5.log 2>&1; tail -1 gpurun_out/fin2/bench_c5.log | cut -c1-150
