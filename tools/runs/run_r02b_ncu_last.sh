# final-build captures: k_generic32 on 4 frames of the whole c4 detector (no tail wave), k_lattice_i8 on the c2 bench shape
mkdir -p gpurun_out/nl
FRAMES=4 PIXELS=1048576 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_generic32" -c 1 -o gpurun_out/nl/gen_c4full -f python tools/time_generic.py > gpurun_out/nl/ncu_gen.log 2>&1; tail -1 gpurun_out/nl/ncu_gen.log
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_lattice_i8 -c 1 -o gpurun_out/nl/i8_c2 -f \
    python tools/profile_case.py c2 --repeat 1 > gpurun_out/nl/ncu_i8_c2.log 2>&1; tail -1 gpurun_out/nl/ncu_i8_c2.log
