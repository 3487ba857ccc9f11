# reductions: new vs v1 kernels, serial (isolated timings) and concurrent; logs under gpurun_out/stats/
mkdir -p gpurun_out/stats
timeout 900 python -m pytest tests -x -q -m gpu -k "xsvs or ring or shell or graph or beta or speckle or parity" > gpurun_out/stats/pytest.log 2>&1; tail -3 gpurun_out/stats/pytest.log
for v in main build/libxpcs_v1stats.so; do
  n=$(basename $v .so)
  for mode in 1 0; do
    env $( [ $v != main ] && echo XPCS_LIB=$v ) XPCS_SERIAL_REDUCTIONS=$mode timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/stats/$n.$mode.log 2>&1
    tail -1 gpurun_out/stats/$n.$mode.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$n serial=$mode', d['value'], d['ms_per_step'], {k: round(v,4) for k,v in d['kernel_ms'].items()})" || tail -5 gpurun_out/stats/$n.$mode.log
  done
done
