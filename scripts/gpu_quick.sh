set -u
timeout 1500 python -m pytest tests/test_gpu_nonlinear.py tests/test_gpu_solver.py -q -x 2>&1 | tail -3
timeout 600 python scripts/nl_bench.py --reps 10 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read())
for k,v in d.items(): print(k, {x: v[x] for x in ('tangent_gdofs','tangent_ms','residual_gdofs') if x in v}, v.get('base_cache_ms'))"
