#!/bin/bash
# solve A/B (DCGS2 dot-sweep rows), BJ tests, ncu of the Krylov kernels mid-solve, tet ncu
set -u
timeout 900 python -m pytest tests/test_gpu_solver.py -q -x -k "block_jacobi" 2>&1 | tail -3
ORTH=dcgs2 bash scripts/ab_solve.sh variants/dcgs16/libldgb200.so variants/dcgs12/libldgb200.so
timeout 600 ncu --set full --clock-control none -k regex:"multidot2|update2|bj_apply" -s 300 -c 3 \
  -o gpurun_out/prof_krylov python scripts/solve_bench.py --n 54 --orth dcgs2 > /dev/null 2>&1
python scripts/ncu_summary.py gpurun_out/prof_krylov.ncu-rep > gpurun_out/ncu_krylov.txt 2>&1; cat gpurun_out/ncu_krylov.txt | head -70
bash scripts/prof_tet.sh > gpurun_out/ncu_tet.txt 2>&1; head -30 gpurun_out/ncu_tet.txt
