#!/bin/bash
# Round-end measurement session: full bench line, reference arm, 2-rank
# bench over gloo, launch list of the bench command, ncu --set full of the
# two fused kernels (summaries + DRAM traffic), config-5 sweep.
set -u
V=${1:-r2}
timeout 900 python bench.py > gpurun_out/bench_${V}.json 2> gpurun_out/bench_${V}.err
tail -c 3000 gpurun_out/bench_${V}.json
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_ref_${V}.json 2>&1
tail -c 600 gpurun_out/bench_ref_${V}.json
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches_${V}.csv python bench.py --steps 2 --warmup 3 --no-solve \
  --no-cpu-baseline --no-nonlinear --no-tet --no-config5 > /dev/null 2>&1
timeout 400 ncu --set full --clock-control none --import-source on \
  -k regex:"plane_kernel|complete_warp" -s 6 -c 2 -o gpurun_out/prof_bench_${V} \
  python bench.py --steps 2 --warmup 3 --no-solve --no-cpu-baseline --no-nonlinear --no-tet --no-config5 > /dev/null 2>&1
python scripts/ncu_summary.py gpurun_out/prof_bench_${V}.ncu-rep > gpurun_out/ncu_summary_${V}.txt 2>&1
python scripts/ncu_traffic.py gpurun_out/prof_bench_${V}.ncu-rep "ncu --set full, profiles/${V}_ncu_summary.txt" > /dev/null 2>&1; cp profiles/traffic.json gpurun_out/traffic_${V}.json
head -45 gpurun_out/ncu_summary_${V}.txt
timeout 600 python scripts/sweep_config5.py > gpurun_out/sweep_config5_${V}.json 2>&1; tail -3 gpurun_out/sweep_config5_${V}.json
