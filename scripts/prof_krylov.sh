#!/bin/bash
# ncu --set full of the config-3 solve's Krylov / block-Jacobi kernels mid-solve
set -u
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"multidot2_all|update2|bj_apply_tiles|finish" \
  -s 400 -c 8 -o gpurun_out/prof_krylov python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-nonlinear \
  --no-tet --no-config5 > gpurun_out/prof_krylov.log 2>&1
python scripts/ncu_summary.py gpurun_out/prof_krylov.ncu-rep > gpurun_out/ncu_krylov.txt 2>&1; cat gpurun_out/ncu_krylov.txt | head -90
