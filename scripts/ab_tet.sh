#!/bin/bash
# tet p=3 matvec (config-3 tet variant) per library build
for lib in paper_2205_07824_b200/lib/libldgb200.so "$@"; do
  LDGB200_LIB=$PWD/$lib timeout 300 python -c "
import sys; sys.path.insert(0, '.')
import bench
r = bench.tet_line(6553.0)
print('$lib', round(r['ms'], 3), round(r['gdofs'], 2))"
done
