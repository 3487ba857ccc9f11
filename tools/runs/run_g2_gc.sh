# one-row g2: frames per staged chunk (GC) 96 / 128 (shipped) / 160 / 192, c2 and c3 shapes alone
mkdir -p gpurun_out/gc
for v in main gc96 gc160 gc192; do
  if [ $v = main ]; then unset XPCS_LIB; else export XPCS_LIB=$PWD/build/libxpcs_$v.so; fi
  timeout 300 python tools/time_g2.py c2 c3 >> gpurun_out/gc/time_g2.log 2>&1
done
unset XPCS_LIB; cat gpurun_out/gc/time_g2.log
