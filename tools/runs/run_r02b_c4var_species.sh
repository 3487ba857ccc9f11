# c4 generic kernel variants (derived fp32 fractions, 4 q per thread) on 4 frames of the whole detector; the
# vectorised species combine: species parity tests + the c3 bench line
mkdir -p gpurun_out/r2d
for v in main derive derive_b4 derive_q4 q4; do
  if [ $v = main ]; then unset XPCS_LIB; else export XPCS_LIB=$PWD/build/libxpcs_$v.so; fi
  FRAMES=4 PIXELS=1048576 timeout 300 python tools/time_generic.py >> gpurun_out/r2d/time_generic.log 2>&1
done
unset XPCS_LIB; cat gpurun_out/r2d/time_generic.log
timeout 1500 python -m pytest -q -m gpu tests -k "species or c3 or c5 or config3 or config5 or volume or step_host" > gpurun_out/r2d/pytest.log 2>&1; tail -2 gpurun_out/r2d/pytest.log
timeout 900 python bench.py > gpurun_out/r2d/bench_c3.log 2>&1; tail -1 gpurun_out/r2d/bench_c3.log | cut -c1-200
