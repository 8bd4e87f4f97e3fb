#!/bin/bash
# exact FP64 operation counts of the pass-1 / pass-2 kernels of the config-3
# bench (ncu), written to gpurun_out/fp64_counts.csv
timeout 300 ncu --metrics smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,gpu__time_duration.sum \
  -k regex:"plane_kernel|complete_warp" -s 6 -c 2 --csv --log-file gpurun_out/fp64_counts.csv \
  python bench.py --steps 2 --warmup 3 --no-solve --no-cpu-baseline --no-nonlinear --no-tet > /dev/null 2>&1
grep -E "dfma|dmul|dadd" gpurun_out/fp64_counts.csv | cut -c1-250 | head
