# XSVS: one-warp / two-warp blocks with a register cap that fits every warp of c5 / c3 in one resident wave
mkdir -p gpurun_out/xw
for v in main x1m15 x1m14 x2m8 x2m7; do
  if [ $v = main ]; then unset XPCS_LIB; else export XPCS_LIB=$PWD/build/libxpcs_$v.so; fi
  timeout 300 python tools/time_xsvs.py c5 c3 >> gpurun_out/xw/time_xsvs.log 2>&1
done
unset XPCS_LIB; cat gpurun_out/xw/time_xsvs.log
