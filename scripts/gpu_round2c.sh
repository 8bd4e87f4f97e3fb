#!/bin/bash
set -u
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_solver.py -q -x -k "tet or tri or simplex or config1 or criterion" 2>&1 | tail -4
bash scripts/ab_tet.sh variants/nodensemma/libldgb200.so
bash scripts/prof_tet.sh > gpurun_out/ncu_tet_mma.txt 2>&1; head -40 gpurun_out/ncu_tet_mma.txt
