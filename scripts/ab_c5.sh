#!/bin/bash
# config-5 A/B of library builds at given orders: ./scripts/ab_c5.sh "4" lib1 lib2 ...
set -u
PS=$1; shift
for lib in paper_2205_07824_b200/lib/libldgb200.so "$@"; do
  LDGB200_LIB=$PWD/$lib timeout 600 python scripts/sweep_config5.py --p $PS 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib', [(r['p'], round(r['gdofs'],1)) for r in d['rows']])"
done
