# round-2 re-entry check: smoke, GPU suite, default bench (c3), c2 bench
mkdir -p gpurun_out/recheck
python -c "import __graft_entry__ as g; g.build(); g.smoke(); print('smoke ok')" > gpurun_out/recheck/smoke.log 2>&1; echo "smoke rc=$?"
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/recheck/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/recheck/pytest.log
timeout 400 python bench.py > gpurun_out/recheck/bench_c3.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/recheck/bench_c3.log | cut -c1-400
timeout 300 python bench.py --config c2 > gpurun_out/recheck/bench_c2.log 2>&1; echo "bench c2 rc=$?"; tail -1 gpurun_out/recheck/bench_c2.log | cut -c1-300
