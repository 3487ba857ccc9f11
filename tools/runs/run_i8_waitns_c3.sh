# c3 under the power cap: try_wait suspend-time hints in the integer engine's barrier waits (alternating runs)
mkdir -p gpurun_out/waitns
for rep in 1 2; do
  for v in base w2k w20k; do
    if [ $v = base ]; then lib=""; else lib="XPCS_LIB=build/libxpcs_$v.so"; fi
    env $lib timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/waitns/$v.$rep.log 2>&1
    tail -1 gpurun_out/waitns/$v.$rep.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', $rep, '%.4e' % d['value'], round(d['ms_per_step'],2), d['clocks']['sm_mhz'], d['roofline']['frac'])" || tail -3 gpurun_out/waitns/$v.$rep.log
  done
done
