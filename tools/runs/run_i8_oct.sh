# integer engine: 8 atoms per producer thread (STS.64, one X + one W warp per group) -- parity of one variant on the
# integer-engine suite, then c3 / c2 bench steps for 4 / 5 / 6 / 8 groups vs the shipped 4 atoms x 4 groups
mkdir -p gpurun_out/oct
XPCS_LIB=$PWD/build/libxpcs_oct6.so timeout 900 python -m pytest -q -m gpu -x tests/test_gpu_i8.py > gpurun_out/oct/pytest_oct6.log 2>&1; tail -2 gpurun_out/oct/pytest_oct6.log
for v in main oct4 oct5 oct6 oct8; do
  if [ $v = main ]; then unset XPCS_LIB; else export XPCS_LIB=$PWD/build/libxpcs_$v.so; fi
  timeout 600 python bench.py --no-e2e --no-cpu-baseline --steps 5 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('c3 $v', d['value'], round(d['ms_per_step'],3), round(d['kernel_ms']['intensity_i8'],3), d['clocks']['sm_mhz'])" >> gpurun_out/oct/sweep.log 2>&1
  timeout 600 python bench.py --config c2 --no-e2e --no-cpu-baseline --steps 20 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('c2 $v', d['value'], round(d['ms_per_step'],4), round(d['kernel_ms']['intensity_i8'],4), d['clocks']['sm_mhz'])" >> gpurun_out/oct/sweep.log 2>&1
done
unset XPCS_LIB; cat gpurun_out/oct/sweep.log
