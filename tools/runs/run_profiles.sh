# round profile refresh: bench lines c1..c5 + reference, c2 launch list, ncu --set full of the i8 kernel (c2)
# outputs in gpurun_out/prof/ (copied into profiles/ by hand)
mkdir -p gpurun_out/prof
for c in c2 c1 c4 c5 c3; do
  st=20; [ $c = c3 ] && st=3; [ $c = c5 ] && st=5
  timeout 1200 python bench.py --config $c --steps $st --warmup 3 > gpurun_out/prof/bench_$c.json.log 2>&1
  tail -1 gpurun_out/prof/bench_$c.json.log > gpurun_out/prof/bench_$c.json
  python -c "import json; d=json.load(open('gpurun_out/prof/bench_$c.json')); print('$c', d['value'], d['ms_per_step'], d['roofline']['frac'], d['e2e']['value'])" || tail -3 gpurun_out/prof/bench_$c.json.log
done
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/prof/bench_reference_c2.log 2>&1; tail -1 gpurun_out/prof/bench_reference_c2.log > gpurun_out/prof/bench_reference_c2.json; cut -c1-300 gpurun_out/prof/bench_reference_c2.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/prof/launches_c2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/prof/ncu_list.log 2>&1
python tools/launch_summary.py gpurun_out/prof/launches_c2.csv "c2 bench --steps 2 --warmup 3 (graph replays), ncu launch list" > gpurun_out/prof/launches_c2_summary.txt; head -12 gpurun_out/prof/launches_c2_summary.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_lattice_i8 -c 1 -o gpurun_out/prof/i8_c2 python tools/profile_case.py c2 --repeat 1 > gpurun_out/prof/ncu_full.log 2>&1; tail -2 gpurun_out/prof/ncu_full.log
python tools/ncu_summary.py gpurun_out/prof/i8_c2.ncu-rep --json gpurun_out/prof/ncu_i8_c2.json > /dev/null 2>&1; head -c 1500 gpurun_out/prof/ncu_i8_c2.json
