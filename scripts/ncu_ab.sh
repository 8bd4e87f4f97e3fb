#!/bin/bash
# kernel-level A/B of library builds with ncu counters (no timing noise):
#   ./scripts/ncu_ab.sh <kernel regex> "<python command>" lib1 lib2 ...
set -u
K=$1; CMD=$2; shift 2
for lib in paper_2205_07824_b200/lib/libldgb200.so "$@"; do
  LDGB200_LIB=$PWD/$lib timeout 600 ncu --metrics gpu__time_duration.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum,smsp__inst_executed.sum \
    --clock-control none -k regex:"$K" -s 2 -c 3 --csv --log-file gpurun_out/ncu_ab.csv $CMD > /dev/null 2>&1
  python -c "
import csv,sys
rows=[r for r in csv.reader(open('gpurun_out/ncu_ab.csv')) if len(r)>10]
h=rows[0]; ki=h.index('Kernel Name'); mi=h.index('Metric Name'); vi=h.index('Metric Value')
from collections import defaultdict
d=defaultdict(list)
for r in rows[1:]: d[(r[ki][:40], r[mi])].append(float(r[vi].replace(',','')))
for k,v in sorted(d.items()): print('$lib'.split('/')[-2], k[0], k[1], round(sum(v)/len(v),1))
"
done
