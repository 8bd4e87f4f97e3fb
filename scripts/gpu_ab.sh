#!/bin/bash
# parity of the default build on the fused-kernel tests, then an A/B of the
# library variants on the config-3 bench, then ncu of pass 1 (default build)
set -u
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -3
bash scripts/ab_libs.sh "$@"
bash scripts/ab_libs.sh "$@"
timeout 400 ncu --set full --clock-control none --import-source on -k regex:"plane_kernel" -s 3 -c 1 \
  -o gpurun_out/prof_p1 python bench.py --steps 2 --warmup 3 --no-solve --no-cpu-baseline --no-nonlinear --no-tet > /dev/null 2>&1
python scripts/ncu_summary.py gpurun_out/prof_p1.ncu-rep > gpurun_out/ncu_p1.txt 2>&1; head -24 gpurun_out/ncu_p1.txt
