#!/bin/bash
# config-3 tet variant (Kuhn tets n=44, p=3) tangent time per library build
set -u
for lib in paper_2205_07824_b200/lib/libldgb200.so "$@"; do
  LDGB200_LIB=$PWD/$lib timeout 600 python -c "
import sys; sys.path.insert(0, '.')
import bench
r = bench.tet_line(6538.6)
print('$lib', round(r['ms'], 3), 'ms', round(r['gdofs'], 2), 'GDOF/s setup', r['setup_s'])
" 2>&1 | tail -1
done
