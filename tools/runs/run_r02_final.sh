# round-2 final check: smoke(), the full GPU suite, the default bench line
mkdir -p gpurun_out/fin
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/fin/smoke.log 2>&1; tail -1 gpurun_out/fin/smoke.log
timeout 2400 python -m pytest tests -q -m gpu > gpurun_out/fin/pytest_gpu.log 2>&1; tail -3 gpurun_out/fin/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/fin/bench_c3.log 2>&1; tail -1 gpurun_out/fin/bench_c3.log | cut -c1-200
