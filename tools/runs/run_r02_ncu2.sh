# ncu --set full of one k_lattice_i8 and one k_lattice_tc launch in a c3-shaped call (32 frames)
ncu --set full --import-source on --clock-control none -k regex:k_lattice_i8 -c 1 -o gpurun_out/r02b_i8_c3 -f \
    python tools/profile_case.py c3 --frames 32 --repeat 1 > gpurun_out/r02b_ncu_i8.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_lattice_tc -c 1 -o gpurun_out/r02b_tc_c3 -f \
    python tools/profile_case.py c3 --frames 32 --repeat 1 > gpurun_out/r02b_ncu_tc.log 2>&1
