# round-2 final check of the final build: smoke(), the full GPU suite, the default bench line (c3), c4 line
mkdir -p gpurun_out/fin3
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/fin3/smoke.log 2>&1; tail -1 gpurun_out/fin3/smoke.log
timeout 2400 python -m pytest tests -q -m gpu > gpurun_out/fin3/pytest_gpu.log 2>&1; tail -3 gpurun_out/fin3/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/fin3/bench_c3.log 2>&1; tail -1 gpurun_out/fin3/bench_c3.log | cut -c1-200
timeout 900 python bench.py --impl reference > gpurun_out/fin3/bench_ref.log 2>&1; tail -1 gpurun_out/fin3/bench_ref.log | cut -c1-200
