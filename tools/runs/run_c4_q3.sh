# c4 generic kernel: 3 q per thread (3 or 2 CTAs per SM) vs the shipped 2 q x 3 CTAs, whole detector, 4 frames
mkdir -p gpurun_out/c4q3
for v in main q3 q3m2; do
  if [ $v = main ]; then unset XPCS_LIB; else export XPCS_LIB=$PWD/build/libxpcs_$v.so; fi
  FRAMES=4 PIXELS=1048576 timeout 300 python tools/time_generic.py >> gpurun_out/c4q3/time_generic.log 2>&1
done
unset XPCS_LIB; cat gpurun_out/c4q3/time_generic.log
