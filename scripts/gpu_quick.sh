set -u
timeout 900 python -m pytest tests/test_gpu_solver.py -k "partitioned" tests/test_gpu_parity.py -q -x 2>&1 | tail -15
timeout 600 python bench.py --no-tet --no-nonlinear --no-solve --no-cpu-baseline > gpurun_out/bench_q.json 2> gpurun_out/bench_q.err
python -c "
import json; d=json.loads(open('gpurun_out/bench_q.json').read().strip().splitlines()[-1]); print(d['value'], d['e2e'])"
