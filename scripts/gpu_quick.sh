set -u
timeout 1200 python -m pytest tests/test_gpu_nonlinear.py tests/test_gpu_solver.py -q -k "1d or line or fd_vs" 2>&1 | tail -15
