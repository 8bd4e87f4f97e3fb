#!/bin/bash
# ncu --set full of the config-5 pencil passes at p = 4 and 5
for P in 4 5; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"fused_kernel|complete" -s 4 -c 2 \
    -o gpurun_out/prof_c5_p$P python scripts/sweep_config5.py --p $P --reps 2 > gpurun_out/prof_c5_p$P.log 2>&1
  python scripts/ncu_summary.py gpurun_out/prof_c5_p$P.ncu-rep > gpurun_out/ncu_c5_p$P.txt 2>&1; head -42 gpurun_out/ncu_c5_p$P.txt
  python scripts/ncu_lines.py gpurun_out/prof_c5_p$P.ncu-rep 20 fused > gpurun_out/ncu_c5_lines_p$P.txt 2>&1
done
