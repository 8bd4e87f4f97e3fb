#!/bin/bash
# A/B timing of operator variants (run under gpurun):
#   ./scripts/ab_pass1.sh label1 "ENV=.. ENV2=.." label2 "..." ...
set -u
run() {  # label, env string
  local label=$1; local envs=$2
  env $envs python bench.py --no-solve --no-cpu-baseline --steps 20 --warmup 5 > gpurun_out/ab_$label.json 2>gpurun_out/ab_$label.err
  python - "$label" <<'PY'
import json, sys
d = json.loads(open(f"gpurun_out/ab_{sys.argv[1]}.json").read().strip().splitlines()[-1])
print(f"{sys.argv[1]:12s} {d['value']:7.2f} GDOF/s  step {d['ms_per_step']*1e3:7.1f} us  pass1 {d['roofline']['ms']*1e3:6.1f} us  pass2 {d['pass2_roofline']['ms']*1e3:6.1f} us")
PY
}
while [ $# -ge 2 ]; do run "$1" "$2"; shift 2; done
