#!/bin/bash
# A/B of library builds on the e2e (host in -> host out) legs of the config-3 bench
set -u
for rep in 1 2; do
for lib in paper_2205_07824_b200/lib/libldgb200.so "$@"; do
  LDGB200_LIB=$PWD/$lib timeout 300 python bench.py --no-solve --no-cpu-baseline --no-nonlinear --no-tet 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); e=d['e2e']; print('$lib', 'value', round(d['value'],1), 'e2e numpy', round(e['value'],2), round(e['ms_per_step'],3), 'ms  pinned', round(e['pinned_torch']['value'],2))"
done; done
nproc; lscpu | grep -i "model name\|^CPU(s)\|Thread\|Socket" | head -5
