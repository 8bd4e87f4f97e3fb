#!/bin/bash
# parity + timing of pass-1 variant builds: each lib in $@ runs the hex p=3
# oracle/golden parity tests, then the config-3 A/B (scripts/ab_libs.sh)
set -u
for lib in "$@"; do
  echo "== $lib"
  LDGB200_LIB=$PWD/$lib timeout 600 python -m pytest tests/test_gpu_parity.py -q -x \
    -k "golden or larger or sheared or at_scale or fused_equals or periodic" 2>&1 | tail -1
done
bash scripts/ab_libs.sh "$@"
bash scripts/ab_libs.sh "$@"
