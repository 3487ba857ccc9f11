# ncu launch list (per-kernel device time) of a short c2 bench for the main build and the v1stats variant
mkdir -p gpurun_out/ncul
for v in main build/libxpcs_v1stats.so; do
  n=$(basename $v .so)
  env $( [ $v != main ] && echo XPCS_LIB=$v ) XPCS_SERIAL_REDUCTIONS=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ncul/$n.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-graph > gpurun_out/ncul/$n.log 2>&1
  python tools/launch_summary.py gpurun_out/ncul/$n.csv "$n" | head -20
done
