# timing experiment: the integer engine with its per-atom step sincos replaced by a cheap placeholder (wrong results,
# fix-up off) vs the main build: how much the producers' setup costs in the c3 / c2 steps
mkdir -p gpurun_out/fs
for v in main fake; do
  L=""; [ $v = fake ] && L=build/var/fake/libxpcs.so
  for c in c3 c2; do
    XPCS_LIB=${L:-paper_2204_13241_b200/lib/libxpcs.so} XPCS_FIXUP=0 timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/fs/$v$c.log 2>&1
    tail -1 gpurun_out/fs/$v$c.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v $c', round(d['ms_per_step'],3), d['clocks']['sm_mhz'], round(d['kernel_ms']['intensity_i8'],3))"
  done
done
