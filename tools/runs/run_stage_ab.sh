for v in main build/libxpcs_stage_old.so main build/libxpcs_stage_old.so; do
env $( [ $v != main ] && echo XPCS_LIB=$v ) timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['kernel_ms']['stage'],4), d['secondary_rooflines']['stage']['ms'], round(d['ms_per_step'],4))"
done
