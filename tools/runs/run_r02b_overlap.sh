# frame-batch overlap (two streams, two buffer sets): parity (new batched test + engine suites), c3 / c2 bench lines
# with and without it (XPCS_BATCH_OVERLAP=0)
mkdir -p gpurun_out/ovl
timeout 1200 python -m pytest -q -m gpu -x tests/test_gpu_volume_species.py tests/test_gpu_i8.py tests/test_gpu_graph.py tests/test_gpu_parity.py > gpurun_out/ovl/pytest.log 2>&1; tail -3 gpurun_out/ovl/pytest.log
for ov in 1 0; do
  XPCS_BATCH_OVERLAP=$ov timeout 900 python bench.py --no-cpu-baseline > gpurun_out/ovl/bench_c3_ov$ov.log 2>&1
  tail -1 gpurun_out/ovl/bench_c3_ov$ov.log | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('c3 ov$ov', d['value'], round(d['ms_per_step'],3), d['e2e']['value'], d['clocks']['sm_mhz'])"
  XPCS_BATCH_OVERLAP=$ov timeout 600 python bench.py --config c2 --no-cpu-baseline > gpurun_out/ovl/bench_c2_ov$ov.log 2>&1
  tail -1 gpurun_out/ovl/bench_c2_ov$ov.log | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('c2 ov$ov', d['value'], round(d['ms_per_step'],4), d['e2e']['value'], d['clocks']['sm_mhz'])"
done
