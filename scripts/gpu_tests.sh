#!/bin/bash
# GPU test suite + bench lines (run under gpurun; outputs in gpurun_out/)
set -u
timeout 1500 python -m pytest tests -m gpu -q --durations=10 > gpurun_out/t_all.txt 2>&1; tail -25 gpurun_out/t_all.txt
timeout 600 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err
tail -c 1500 gpurun_out/bench_full.json
# two ranks sharing the GPU through gloo (exercises the self-launch, the
# partitioned matvec with face-node halos and the distributed solve)
LDG_DIST_BACKEND=gloo timeout 600 python bench.py --gpus 2 --steps 3 --warmup 3 --elems 24 \
  --no-tet --no-nonlinear --no-cpu-baseline > gpurun_out/bench_2rank.json 2> gpurun_out/bench_2rank.err
tail -c 1500 gpurun_out/bench_2rank.json; tail -5 gpurun_out/bench_2rank.err
