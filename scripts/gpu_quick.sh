set -u
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_solver.py -q -x -k "partitioned" 2>&1 | tail -15
