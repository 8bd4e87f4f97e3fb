#!/bin/bash
# ncu --set full of the generated NS3D tangent kernel (config-4 shape, n=16)
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"nl_tangent" -s 2 -c 1 \
  -o gpurun_out/prof_nl python scripts/nl_profile.py 16 > gpurun_out/prof_nl.log 2>&1
python scripts/ncu_summary.py gpurun_out/prof_nl.ncu-rep
python scripts/ncu_lines.py gpurun_out/prof_nl.ncu-rep 40
