#!/bin/bash
# A/B of the plane kernel's diagonal-C and general-C variants: bench value and
# pass-1 time for each, ncu --set full of the pass-1 kernel (outputs in gpurun_out/)
set -u
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_solver.py -m gpu -q -x > gpurun_out/t.txt 2>&1; tail -3 gpurun_out/t.txt
for d in 1 0; do
LDG_CDIAG=$d timeout 300 python bench.py --no-solve --no-cpu-baseline --no-nonlinear --no-tet 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('CDIAG', $d, d['value'], d['roofline']['ms'], d['roofline']['kernel'])"
LDG_CDIAG=$d timeout 300 ncu --set full --clock-control none --import-source on \
  -k regex:"plane_kernel" -s 3 -c 1 -o gpurun_out/prof_plane_d$d \
  python bench.py --steps 2 --warmup 3 --no-solve --no-cpu-baseline --no-nonlinear --no-tet > /dev/null 2>&1
python scripts/ncu_summary.py gpurun_out/prof_plane_d$d.ncu-rep > gpurun_out/sum_d$d.txt 2>&1
done
cat gpurun_out/sum_d1.txt
