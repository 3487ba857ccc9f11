# xsvs_contrast timing for the main build and build/var/* variants (tools/build_variants.sh)
mkdir -p gpurun_out/xv
timeout 300 python tools/time_xsvs.py > gpurun_out/xv/main.json 2>&1; cat gpurun_out/xv/main.json | tail -1
for v in build/var/*/; do
  n=$(basename $v)
  XPCS_LIB=$v/libxpcs.so timeout 300 python tools/time_xsvs.py > gpurun_out/xv/$n.json 2>&1; tail -1 gpurun_out/xv/$n.json
done
if [ -n "$XV_NCU" ]; then
  XPCS_LIB=build/var/$XV_NCU/libxpcs.so ncu --set full --clock-control none --import-source on -k regex:xsvs_warp2 -c 1 -o gpurun_out/xv/ncu_$XV_NCU python tools/time_xsvs.py c5 > gpurun_out/xv/ncu.log 2>&1; echo ncu $?
fi
