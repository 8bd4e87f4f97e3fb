set -u
timeout 600 python -m pytest tests/test_gpu_solver.py -q -x -k "mgs-poisson1d" 2>&1 | grep -E "Error|assert|error|^E " | head -20
