for v in default pe0; do
  if [ $v = default ]; then L=""; else L="XPCS_LIB=build/libxpcs_$v.so"; fi
  env $L ncu --set full --import-source on -k regex:k_generic32 -c 1 -o gpurun_out/r02_c4_$v -f python tools/profile_case.py c4 --frames 1 --pixels 262144 --repeat 1 > gpurun_out/ncu_c4_$v.log 2>&1
done
