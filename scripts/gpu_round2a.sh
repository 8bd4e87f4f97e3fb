#!/bin/bash
# A/B of the pass-1 DMMA variants + ncu of the generated NS tangent (config 4)
set -u
bash scripts/ab_libs.sh variants/nodmma/libldgb200.so variants/dmma1/libldgb200.so variants/dmma2/libldgb200.so
bash scripts/prof_nl.sh > gpurun_out/ncu_nl.txt 2>&1; head -60 gpurun_out/ncu_nl.txt
