#!/bin/bash
# One GPU session: GPU tests, full bench line, launch list, ncu --set full of
# the two fused kernels (run under gpurun; outputs in gpurun_out/)
set -u
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/t_all.txt 2>&1; tail -3 gpurun_out/t_all.txt
timeout 900 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err
tail -c 400 gpurun_out/bench_full.json
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-solve \
  --no-cpu-baseline --no-nonlinear --no-tet > /dev/null 2>&1
timeout 400 ncu --set full --clock-control none --import-source on \
  -k regex:"plane_kernel|complete_warp" -s 6 -c 2 -o gpurun_out/prof_bench \
  python bench.py --steps 2 --warmup 3 --no-solve --no-cpu-baseline --no-nonlinear --no-tet > /dev/null 2>&1
python scripts/ncu_summary.py gpurun_out/prof_bench.ncu-rep > gpurun_out/ncu_summary.txt 2>&1
ls -la gpurun_out | tail -5
