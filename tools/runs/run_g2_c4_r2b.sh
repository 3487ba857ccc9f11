# g2: one block row per <= 256 lags (balanced groups of 8 per warp) -- parity + timing; c4: I2FP turns variants
mkdir -p gpurun_out/g2c4
timeout 900 python -m pytest -q -m gpu tests/test_gpu_parity.py -k g2 tests/test_gpu_g2_stream.py tests/test_gpu_golden.py > gpurun_out/g2c4/pytest.log 2>&1; tail -2 gpurun_out/g2c4/pytest.log
timeout 300 python tools/time_g2.py c2 c3 > gpurun_out/g2c4/time_g2.log 2>&1; tail -2 gpurun_out/g2c4/time_g2.log
for v in main i2f i2f_q4 i2f_b4; do
  if [ $v = main ]; then unset XPCS_LIB; else export XPCS_LIB=$PWD/build/libxpcs_$v.so; fi
  timeout 300 python tools/time_generic.py >> gpurun_out/g2c4/time_generic.log 2>&1
done
unset XPCS_LIB; cat gpurun_out/g2c4/time_generic.log
