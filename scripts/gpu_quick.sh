set -u
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "variants" 2>&1 | tail -5
bash scripts/sanitize.sh
