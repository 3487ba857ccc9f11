# round-2 re-entry check: smoke(), the full GPU suite, the default bench line (c3) and c2
mkdir -p gpurun_out/r2b
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r2b/smoke.log 2>&1; tail -1 gpurun_out/r2b/smoke.log
timeout 2400 python -m pytest tests -q -m gpu -x > gpurun_out/r2b/pytest_gpu.log 2>&1; tail -3 gpurun_out/r2b/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/r2b/bench_c3.log 2>&1; tail -1 gpurun_out/r2b/bench_c3.log | cut -c1-300
timeout 600 python bench.py --workload c2 > gpurun_out/r2b/bench_c2.log 2>&1; tail -1 gpurun_out/r2b/bench_c2.log | cut -c1-300
