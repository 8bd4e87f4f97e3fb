#!/bin/bash
# one-launch operator (plane_kernel<.., FUSED>): bitwise tests, A/B on config 3, ncu
set -u
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "one_launch" > gpurun_out/t_fused.txt 2>&1; tail -3 gpurun_out/t_fused.txt
grep -q "passed" gpurun_out/t_fused.txt && ! grep -q "failed" gpurun_out/t_fused.txt || exit 1
for f in 0 1 0 1; do
  timeout 300 python bench.py --no-solve --no-cpu-baseline --no-nonlinear --no-tet --fused $f 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('fused=$f', round(d['value'],2), 'step_us', round(d['ms_per_step']*1e3,1), 'e2e', round(d['e2e']['value'],2))"
done
timeout 300 ncu --set full --clock-control none --import-source on -k regex:"plane_kernel" -s 3 -c 1 \
  -o gpurun_out/prof_fused python bench.py --steps 2 --warmup 3 --no-solve --no-cpu-baseline --no-nonlinear --no-tet --fused 1 > /dev/null 2>&1
python scripts/ncu_summary.py gpurun_out/prof_fused.ncu-rep > gpurun_out/ncu_fused.txt 2>&1; head -25 gpurun_out/ncu_fused.txt
