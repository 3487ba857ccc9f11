# final round-2 captures: ncu --set full of one k_lattice_i8 and one k_lattice_tc launch (c3 shape, 32 frames), and the
# launch list of the default bench command (c3)
ncu --set full --import-source on --clock-control none -k regex:k_lattice_i8 -c 1 -o gpurun_out/r02c_i8_c3 -f \
    python tools/profile_case.py c3 --frames 32 --repeat 1 > gpurun_out/r02c_ncu_i8.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_lattice_tc -c 1 -o gpurun_out/r02c_tc_c3 -f \
    python tools/profile_case.py c3 --frames 32 --repeat 1 > gpurun_out/r02c_ncu_tc.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02c_launches_c3.csv \
    python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/r02c_ncu_list.log 2>&1
