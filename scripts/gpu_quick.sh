set -u
timeout 900 python -m pytest tests/test_gpu_nonlinear.py -q -x -k "curved" 2>&1 | tail -15
timeout 900 python -m pytest tests/test_gpu_solver.py -q -x -k "curved" 2>&1 | tail -15
