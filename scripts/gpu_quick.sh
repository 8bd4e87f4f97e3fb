set -u
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -4
bash scripts/ab_tet.sh variants/nodensemma/libldgb200.so
timeout 600 python scripts/nl_bench.py --reps 10 2>&1 | tail -2
bash scripts/prof_tet.sh > gpurun_out/ncu_tet_mma.txt 2>&1; grep -E "=====|duration|wavefronts|conflicts|issue_active|fp64" gpurun_out/ncu_tet_mma.txt | head -24
