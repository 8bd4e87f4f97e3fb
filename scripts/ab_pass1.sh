#!/bin/bash
# A/B timing of the pass-1 kernel variants (run under gpurun)
set -u
run() {  # label, env...
  local label=$1; shift
  env "$@" python bench.py --no-solve --no-cpu-baseline --steps 20 --warmup 5 > gpurun_out/ab_$label.json 2>gpurun_out/ab_$label.err
  python - "$label" <<'PY'
import json, sys
d = json.loads(open(f"gpurun_out/ab_{sys.argv[1]}.json").read().strip().splitlines()[-1])
print(f"{sys.argv[1]:12s} {d['value']:7.2f} GDOF/s  step {d['ms_per_step']*1e3:7.1f} us  pass1 {d['roofline']['ms']*1e3:6.1f} us  pass2 {d['pass2_roofline']['ms']*1e3:6.1f} us")
PY
}
run plane LDG_PASS1_VARIANT=plane
[ -f paper_2205_07824_b200/lib/variants/libldgb200_minb2.so ] && run plane_minb2 LDGB200_LIB=paper_2205_07824_b200/lib/variants/libldgb200_minb2.so
run pencil LDG_PASS1_VARIANT=pencil
