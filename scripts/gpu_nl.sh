#!/bin/bash
# generated kernels: face batching parity + launch-shape A/B on config 4
set -u
timeout 1200 python -m pytest tests/test_gpu_nonlinear.py tests/test_gpu_diagnostics.py -q -x > gpurun_out/t_nl.txt 2>&1; tail -3 gpurun_out/t_nl.txt
timeout 1200 python scripts/nl_ab.py 128,6,3 128,2,3 128,2,4 128,3,4 128,1,4 64,2,5 64,2,6 > gpurun_out/nl_ab.jsonl 2> gpurun_out/nl_ab.err
cat gpurun_out/nl_ab.jsonl; tail -3 gpurun_out/nl_ab.err
