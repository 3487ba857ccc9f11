for v in main build/libxpcs_nosts.so main build/libxpcs_nosts.so; do for f in 0 2; do
env $( [ $v != main ] && echo XPCS_LIB=$v ) XPCS_I8_DEBUG=$f timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v dbg=$f', round(d['kernel_ms']['intensity_main'],4))"
done; done
