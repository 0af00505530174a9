#!/bin/bash
# A/B timing of rollout variants on the GPU box: tools/ab.sh "<env settings>" ...
# prints workload, env, step ms, rollout ms, roofline frac for cfg1 / cfg3 / HBM cartpole 2^20.
out=${OUT:-gpurun_out/ab.txt}
for envs in "$@"; do
  for wl in "--workload cfg1" "--workload cfg3" "--workload cfg1 --noise hbm --samples 1048576" ${EXTRA_WL:+"$EXTRA_WL"}; do
    line=$(env $envs python bench.py $wl --steps ${STEPS:-10} --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1)
    python - "$envs" "$wl" "$line" >> $out <<'PY'
import json, sys
envs, wl, line = sys.argv[1:4]
try:
    d = json.loads(line); r = d["roofline"]
    h = r.get("hbm", {})
    print(f"{wl:48s} {envs:24s} step {d['ms_per_step']*1e3:9.2f} us  rollout {r['kernel_ms']*1e3:9.2f} us  fp32 {r['frac']:.3f}  hbm {h.get('frac', 0):.3f}")
except Exception as e:
    print(f"{wl:48s} {envs:24s} FAILED {line[-300:]}")
PY
  done
done
