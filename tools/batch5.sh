#!/bin/bash
# drop-in call: one graph launch (default) vs three stream launches (JM_DROPIN_DIRECT=1)
o=gpurun_out/b5; mkdir -p $o
for wl in cfg0 cfg1 cfg2; do
  for envs in "JM_X=0" "JM_DROPIN_DIRECT=1"; do
    for rep in 1 2; do
    echo "$wl $envs $(env $envs python bench.py --workload $wl --steps 200 --warmup 20 --no-cpu-baseline 2>&1 | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print("step_us %.2f e2e_us %.2f" % (d["ms_per_step"]*1e3, d["e2e"]["ms_per_step"]*1e3))')" >> $o/e2e.txt
    done
  done
done
python tools/e2e_split.py > $o/e2e_split.txt 2>&1
JM_DROPIN_DIRECT=1 python tools/e2e_split.py > $o/e2e_split_direct.txt 2>&1
cat $o/e2e.txt; cat $o/e2e_split.txt $o/e2e_split_direct.txt
