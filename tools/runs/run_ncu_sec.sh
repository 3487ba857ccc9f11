mkdir -p gpurun_out/sec
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_g2|k_xsvs_warp2|k_shell_mean|k_stage_lattice32|k_xsvs_final" -c 6 -o gpurun_out/sec/sec python tools/profile_case.py c2 --repeat 1 > gpurun_out/sec/ncu.log 2>&1; tail -2 gpurun_out/sec/ncu.log
python tools/ncu_summary.py gpurun_out/sec/sec.ncu-rep --json gpurun_out/sec/sec.json > /dev/null 2>&1; ls -la gpurun_out/sec
