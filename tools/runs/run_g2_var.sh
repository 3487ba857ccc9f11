# xpcs_g2 timing for the main build and build/var/* variants (tools/build_variants.sh)
mkdir -p gpurun_out/gv
timeout 300 python tools/time_g2.py > gpurun_out/gv/main.json 2>&1; tail -1 gpurun_out/gv/main.json
for v in build/var/*/; do
  n=$(basename $v)
  XPCS_LIB=$v/libxpcs.so timeout 300 python tools/time_g2.py > gpurun_out/gv/$n.json 2>&1; tail -1 gpurun_out/gv/$n.json
done
if [ -n "$GV_NCU" ]; then
  XPCS_LIB=build/var/$GV_NCU/libxpcs.so ncu --set full --clock-control none --import-source on -k regex:k_g2 -c 1 -o gpurun_out/gv/ncu_$GV_NCU python tools/time_g2.py c3 > gpurun_out/gv/ncu.log 2>&1; echo ncu $?
fi
