# i8 chunking / tail-split calibration on c2 (kernel ms per configuration); logs under gpurun_out/i8chunk/
mkdir -p gpurun_out/i8chunk
run() { n=$1; shift; env "$@" timeout 300 python bench.py --config c2 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/i8chunk/$n.log 2>&1;
  tail -1 gpurun_out/i8chunk/$n.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$n', d['ms_per_step'], d['kernel_ms'])" || tail -3 gpurun_out/i8chunk/$n.log; }
if [ -z "$SKIP_TESTS" ]; then timeout 900 python -m pytest tests/test_gpu_i8.py tests/test_gpu_parity.py -x -q -m gpu > gpurun_out/i8chunk/pytest.log 2>&1; tail -3 gpurun_out/i8chunk/pytest.log; fi
run default XPCS_X=1
run notail XPCS_I8_TAILSPLIT=0
for c in ${CHUNKS:-32000 16000 10688 8000 6400 4576 3200}; do run ch$c XPCS_CHUNK_ATOMS=$c; done
