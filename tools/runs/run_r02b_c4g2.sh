# after the I2FP generic kernel and the one-row g2: generic parity (incl. the c4 full-size sampled test), c3 bench,
# c4 bench line, ncu --set full of k_g2 (c3 shape) and k_generic32 (c4 slice)
mkdir -p gpurun_out/r2c
timeout 1200 python -m pytest -q -m gpu tests/test_gpu_parity.py tests/test_gpu_fullsize.py -k "generic or c4 or config4 or g2" > gpurun_out/r2c/pytest.log 2>&1; tail -2 gpurun_out/r2c/pytest.log
timeout 900 python bench.py > gpurun_out/r2c/bench_c3.log 2>&1; tail -1 gpurun_out/r2c/bench_c3.log | cut -c1-200
timeout 900 python bench.py --config c4 --steps 3 --warmup 3 --no-e2e > gpurun_out/r2c/bench_c4.log 2>&1; tail -1 gpurun_out/r2c/bench_c4.log | cut -c1-200
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_g2" -c 1 -o gpurun_out/r2c/g2_c3 python tools/time_g2.py c3 > gpurun_out/r2c/ncu_g2.log 2>&1; tail -1 gpurun_out/r2c/ncu_g2.log
FRAMES=1 PIXELS=262144 timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_generic32" -c 1 -o gpurun_out/r2c/gen_c4 python tools/time_generic.py > gpurun_out/r2c/ncu_gen.log 2>&1; tail -1 gpurun_out/r2c/ncu_gen.log
