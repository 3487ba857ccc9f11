# integer engine on c2: full / MMA-only (skip generation) / production-only (skip MMA) / neither
mkdir -p gpurun_out/i8dbg
for f in 0 2 4 6; do
  XPCS_I8_DEBUG=$f timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/i8dbg/$f.log 2>&1
  tail -1 gpurun_out/i8dbg/$f.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('dbg=$f', d['kernel_ms']['intensity_main'], d['roofline']['vs_mma_issue_rate']['frac'])" || tail -3 gpurun_out/i8dbg/$f.log
done
