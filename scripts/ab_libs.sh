#!/bin/bash
# A/B of library builds (variants/*/libldgb200.so, built with different -D
# flags) on the config-3 bench: value, pass-1 and pass-2 times per build
set -u
for lib in paper_2205_07824_b200/lib/libldgb200.so "$@"; do
  LDGB200_LIB=$PWD/$lib timeout 300 python bench.py --no-solve --no-cpu-baseline --no-nonlinear --no-tet 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib', round(d['value'],2), 'p1', round(d['roofline']['ms']*1e3,1), 'p2', round(d['pass2_roofline']['ms']*1e3,1))"
done
