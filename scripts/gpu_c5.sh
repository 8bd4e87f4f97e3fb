#!/bin/bash
# config-5 plane kernels (hex p = 1, 2): parity tests, sweep, ncu of pass 1 at p = 1 and 2
set -u
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "p1_p2 or sheared or variants or larger or periodic or golden or nan or partitioned_native" \
  > gpurun_out/t_c5.txt 2>&1; tail -5 gpurun_out/t_c5.txt
timeout 600 python scripts/sweep_config5.py > gpurun_out/sweep_c5.json 2>&1; tail -c 2500 gpurun_out/sweep_c5.json
for P in 1 2; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"plane_kernel_g|complete" -s 4 -c 2 \
    -o gpurun_out/prof_c5_p$P python scripts/sweep_config5.py --p $P --reps 2 > gpurun_out/prof_c5_p$P.log 2>&1
  python scripts/ncu_summary.py gpurun_out/prof_c5_p$P.ncu-rep > gpurun_out/ncu_c5_p$P.txt 2>&1
  head -40 gpurun_out/ncu_c5_p$P.txt
done
