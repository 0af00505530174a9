#!/bin/bash
# A/B batch: MUFU quadrotor sincos (main), cost2 + HBM depth 3 (v2), SPT=2 at cfg1, timeline
o=gpurun_out/b2; mkdir -p $o
JM_GATE_REPORT=$o/gate.jsonl python -m pytest tests -m gpu -x -q > $o/pytest_gpu.txt 2>&1; echo "pytest exit $?" >> $o/pytest_gpu.txt
export OUT=$o/ab.txt STEPS=10
EXTRA_WL="--workload cfg3 --noise hbm" bash tools/ab.sh "JM_X=0" "JM_LIB=scratch/libjm_v2.so"
for wl in cfg2 cfg0; do
  for envs in "JM_X=0" "JM_LIB=scratch/libjm_v2.so"; do
    echo "$wl $envs $(env $envs python bench.py --workload $wl --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"]*1e3, d["roofline"]["kernel_ms"]*1e3)')" >> $o/ab.txt
  done
done
echo "cfg1 JM_SPT=2 $(JM_SPT=2 python bench.py --workload cfg1 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"]*1e3, d["roofline"]["kernel_ms"]*1e3, d["roofline"]["kernel"])')" >> $o/ab.txt
JM_TIMELINE=1 python tools/timeline.py cfg1 40 > $o/timeline_cfg1.txt 2>&1
JM_TIMELINE=1 JM_SPT=2 python tools/timeline.py cfg1 40 > $o/timeline_cfg1_spt2.txt 2>&1
JM_TIMELINE=1 python tools/timeline.py cfg0 40 > $o/timeline_cfg0.txt 2>&1
cat $o/ab.txt
