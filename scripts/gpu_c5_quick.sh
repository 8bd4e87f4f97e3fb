#!/bin/bash
# plane_kernel_g quick check: p = 1, 2 parity subset + config-5 rows p = 1, 2
set -u
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "p1_p2 or sheared or variants or larger or periodic or golden" \
  > gpurun_out/t_c5q.txt 2>&1; tail -3 gpurun_out/t_c5q.txt
timeout 600 python scripts/sweep_config5.py --p 1,2 > gpurun_out/sweep_c5q.json 2>&1; tail -c 1200 gpurun_out/sweep_c5q.json
