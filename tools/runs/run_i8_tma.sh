timeout 900 python -m pytest tests/test_gpu_i8.py tests/test_gpu_parity.py -x -q -m gpu 2>&1 | tail -2
VARIANTS="main build/libxpcs_notma.so build/libxpcs_tma7.so main" bash tools/runs/run_i8_sweep.sh
