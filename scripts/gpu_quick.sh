set -u
timeout 600 python scripts/nl_bench.py --reps 10 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read())
for k,v in d.items(): print(k, {x: v.get(x) for x in ('tangent_gdofs','tangent_ms','tangent_uncached_ms','base_cache_ms','residual_gdofs')}, v['attrs'].get('nl_tangent_cached'))"
timeout 600 python -m pytest tests/test_gpu_nonlinear.py -q -x -k "ns3d" 2>&1 | tail -2
