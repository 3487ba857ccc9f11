# c3 power attribution of the integer engine: the same build with production skipped (XPCS_I8_DEBUG=2) or MMAs
# skipped (=4); fix-up off (the skipped variants produce garbage intensities).  Step time and SM clock per variant.
mkdir -p gpurun_out/pw
for d in 0 2 4; do
  XPCS_LIB=build/var/exp/libxpcs.so XPCS_I8_DEBUG=$d XPCS_FIXUP=0 timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/pw/d$d.log 2>&1
  tail -1 gpurun_out/pw/d$d.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('dbg $d', round(d['ms_per_step'],1), d['clocks'], round(d['kernel_ms']['intensity_i8'],1))"
done
