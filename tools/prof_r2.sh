#!/bin/bash
# round-2 ncu captures (one rollout launch each): cfg1, cfg3, cartpole 2^20 HBM, cfg0, cfg2
mkdir -p gpurun_out/prof
run() { # name, counters key, bench args
  name=$1; shift; key=$1; shift
  B="python bench.py --steps 2 --warmup 1 --profile --no-cpu-baseline --no-e2e $*"
  $B > gpurun_out/prof/plain_$name.log 2>&1 || return
  ncu --set full --clock-control none --import-source on -k regex:rollout_ -s 2 -c 1 -o gpurun_out/prof/$name $B > gpurun_out/prof/ncu_$name.log 2>&1
  python tools/ncu_summary.py gpurun_out/prof/$name.ncu-rep > gpurun_out/prof/$name.summary.txt 2>&1
  python tools/ncu_stalls.py gpurun_out/prof/$name.ncu-rep 60 > gpurun_out/prof/$name.stalls.txt 2>&1
  python tools/ncu_lines.py gpurun_out/prof/$name.ncu-rep 70 > gpurun_out/prof/$name.lines.txt 2>&1 || true
  python tools/ncu_counters.py gpurun_out/prof/$name.ncu-rep $key "profiles/${PROF_DIR:-r2}/$name.summary.txt" gpurun_out/prof/kernel_counters.json >> gpurun_out/prof/counters.log 2>&1
}
run cfg1 cfg1/f32/philox/K=65536 --workload cfg1
run cfg3 cfg3/f32/philox/K=1048576 --workload cfg3
run hbm_cart1M cfg1/f32/hbm/K=1048576 --workload cfg1 --noise hbm --samples 1048576
run cfg0 cfg0/f32/philox/K=1024 --workload cfg0
run cfg2 cfg2/f32/philox/K=8192 --workload cfg2
ls -la gpurun_out/prof; mkdir -p /tmp/reps && mv gpurun_out/prof/*.ncu-rep /tmp/reps/ 2>/dev/null || true
cp gpurun_out/prof/kernel_counters.json profiles/kernel_counters.json
