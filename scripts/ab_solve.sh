#!/bin/bash
# solve time (config 3) per library build: bash scripts/ab_solve.sh variants/x/libldgb200.so ...
for lib in paper_2205_07824_b200/lib/libldgb200.so "$@"; do
  echo "$lib"; LDGB200_LIB=$PWD/$lib timeout 300 python scripts/solve_bench.py --n 54 --orth ${ORTH:-cgs2} 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read())['gpu']; print({k: d[k] for k in ('precond_build_s','solve_s','warm_precond_build_s','warm_solve_s','gmres')})"
done
