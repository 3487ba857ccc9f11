# c4 generic kernel: 3 vs 4 CTAs per SM, shift/OR vs I2FP turn conversion, on 4 frames of the whole detector
mkdir -p gpurun_out/c4
for v in main b4 i2f i2f_b4; do
  if [ $v = main ]; then unset XPCS_LIB; else export XPCS_LIB=$PWD/build/libxpcs_$v.so; fi
  FRAMES=4 PIXELS=1048576 timeout 300 python tools/time_generic.py >> gpurun_out/c4/time_generic.log 2>&1
done
unset XPCS_LIB; cat gpurun_out/c4/time_generic.log
