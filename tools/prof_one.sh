#!/bin/bash
# one ncu --set full capture of the rollout kernel of a workload: tools/prof_one.sh <name> <bench args...>
name=$1; shift
mkdir -p gpurun_out/prof1
B="python bench.py --steps 2 --warmup 1 --profile --no-cpu-baseline --no-e2e $*"
$B > gpurun_out/prof1/plain_$name.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:rollout_ -s 2 -c 1 -o gpurun_out/prof1/$name $B > gpurun_out/prof1/ncu_$name.log 2>&1
python tools/ncu_summary.py gpurun_out/prof1/$name.ncu-rep > gpurun_out/prof1/$name.summary.txt 2>&1
python tools/ncu_lines.py gpurun_out/prof1/$name.ncu-rep 60 > gpurun_out/prof1/$name.lines.txt 2>&1 || true
cat gpurun_out/prof1/$name.summary.txt; head -50 gpurun_out/prof1/$name.lines.txt
