timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x 2>&1 | tail -2
bash scripts/ab_libs.sh variants/nopipe/libldgb200.so
bash scripts/ab_libs.sh
