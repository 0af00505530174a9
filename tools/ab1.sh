#!/bin/bash
# repeated A/B of one workload: tools/ab1.sh "<bench args>" "<env A>" "<env B>" ... (3 rounds, interleaved)
args=$1; shift
for round in 1 2 3; do
  for envs in "$@"; do
    line=$(env $envs python bench.py $args --steps ${STEPS:-30} --warmup 5 --no-cpu-baseline --no-e2e 2>&1 | tail -1)
    python - "$envs" "$line" <<'PY'
import json, sys
envs, line = sys.argv[1:3]
try:
    d = json.loads(line); r = d["roofline"]
    print(f"{envs:28s} step {d['ms_per_step']*1e3:9.2f} us  rollout {r['kernel_ms']*1e3:9.2f} us")
except Exception:
    print(f"{envs:28s} FAILED {line[-200:]}")
PY
  done
done
