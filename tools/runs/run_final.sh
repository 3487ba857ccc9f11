mkdir -p gpurun_out/final
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/final/pytest.log 2>&1; tail -2 gpurun_out/final/pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final/smoke.log 2>&1; tail -1 gpurun_out/final/smoke.log
bash tools/runs/run_profiles.sh > gpurun_out/final/profiles.log 2>&1; grep -E "^c[1-5] " gpurun_out/final/profiles.log
