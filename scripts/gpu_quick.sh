set -u
LDG_DIST_BACKEND=gloo timeout 900 python bench.py --gpus 2 --steps 3 --warmup 3 --elems 24 \
  --no-tet --no-nonlinear --no-cpu-baseline > gpurun_out/bench_2rank.json 2> gpurun_out/bench_2rank.err
tail -c 1200 gpurun_out/bench_2rank.json; tail -3 gpurun_out/bench_2rank.err
