#!/bin/bash
# hex p = 1 thread-per-element pass 1: parity subset, config-5 row, ncu
set -u
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "p1_p2 or sheared or variants or larger or periodic" \
  > gpurun_out/t_p1.txt 2>&1; tail -3 gpurun_out/t_p1.txt
timeout 600 python scripts/sweep_config5.py --p 1,2 > gpurun_out/sweep_p1.json 2>&1; tail -c 900 gpurun_out/sweep_p1.json
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"elem_kernel_p1|complete" -s 4 -c 2 \
  -o gpurun_out/prof_p1 python scripts/sweep_config5.py --p 1 --reps 2 > gpurun_out/prof_p1.log 2>&1
python scripts/ncu_summary.py gpurun_out/prof_p1.ncu-rep > gpurun_out/ncu_p1.txt 2>&1; head -40 gpurun_out/ncu_p1.txt
