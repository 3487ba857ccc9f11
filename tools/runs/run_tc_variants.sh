# timing/parity sweep over libxpcs variants (XPCS_LIB); logs under gpurun_out/tcvar/
mkdir -p gpurun_out/tcvar
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_volume_species.py -x -q -m gpu > gpurun_out/tcvar/pytest.log 2>&1
tail -5 gpurun_out/tcvar/pytest.log
for v in ${VARIANTS:-""}; do
  n=$(basename "${v:-main}" .so)
  for c in c2 c3; do
    e=""; [ $c = c2 ] && e="--engine tensor"
    env ${v:+XPCS_LIB=$v} timeout 300 python bench.py $e --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/tcvar/$n.$c.log 2>&1
    echo "$n $c $(tail -1 gpurun_out/tcvar/$n.$c.log | cut -c1-200)"
  done
done
