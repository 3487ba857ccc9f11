# split-FP16 engine on c2: full / MMA-only (skip generation) / production-only (skip MMA) / no drain
mkdir -p gpurun_out/tcdbg
for f in 0 2 4 8 6; do
  XPCS_TC_DEBUG=$f timeout 300 python bench.py --engine tensor --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/tcdbg/$f.log 2>&1
  tail -1 gpurun_out/tcdbg/$f.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('dbg=$f', d['kernel_ms']['intensity_main'], d['roofline']['frac'], d['roofline'].get('vs_mma_issue_rate'))" || tail -3 gpurun_out/tcdbg/$f.log
done
