mkdir -p gpurun_out/ncui8
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_lattice_i8 --launch-skip 1 -c 1 -o gpurun_out/ncui8/i8_c2_direct python tools/profile_case.py c2 --repeat 1 > gpurun_out/ncui8/ncu.log 2>&1; tail -2 gpurun_out/ncui8/ncu.log
python tools/ncu_summary.py gpurun_out/ncui8/i8_c2_direct.ncu-rep --json gpurun_out/ncui8/i8_c2_direct.json > /dev/null 2>&1; head -c 2500 gpurun_out/ncui8/i8_c2_direct.json
