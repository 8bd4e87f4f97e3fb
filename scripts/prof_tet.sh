#!/bin/bash
# ncu --set full of the dense simplex kernels on the config-3 tet variant (n=24 to keep it short)
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"mixed_dense|flux_dense" -s 2 -c 2 \
  -o gpurun_out/prof_tet python -c "
import sys; sys.path.insert(0, '.')
import bench, torch
print(bench.tet_line(6553.0, n=24, reps=2))
" > gpurun_out/prof_tet.log 2>&1
python scripts/ncu_summary.py gpurun_out/prof_tet.ncu-rep
