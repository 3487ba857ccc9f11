# integer engine time attribution on c2 (results of the debug runs are invalid by construction)
for d in 0 2 4 6; do
  XPCS_LIB=build/libxpcs_exp.so XPCS_I8_DEBUG=$d XPCS_FIXUP=0 python bench.py --config c2 --no-e2e --no-cpu-baseline --steps 10 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('dbg', $d, round(d['kernel_ms']['intensity_i8'],4))" >> gpurun_out/attr.log
done
