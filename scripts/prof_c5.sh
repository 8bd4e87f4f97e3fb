#!/bin/bash
# ncu --set full of the config-5 pencil pass-1 / pass-2 kernels at p (default 4)
P=${1:-4}
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"fused_kernel|complete_kernel" -s 4 -c 2 \
  -o gpurun_out/prof_c5 python scripts/sweep_config5.py --p $P --reps 2 > gpurun_out/prof_c5.log 2>&1
python scripts/ncu_summary.py gpurun_out/prof_c5.ncu-rep
python scripts/ncu_lines.py gpurun_out/prof_c5.ncu-rep 25 fused
