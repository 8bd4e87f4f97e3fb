set -u
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
ORTH=dcgs2 bash scripts/ab_solve.sh
