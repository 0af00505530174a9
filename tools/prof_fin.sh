#!/bin/bash
# ncu --set full capture of the finalize kernel of the cfg1 bench step
mkdir -p gpurun_out/proffin
B="python bench.py --steps 2 --warmup 1 --profile --no-cpu-baseline --no-e2e --workload cfg1"
$B > gpurun_out/proffin/plain.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:finalize_ -s 2 -c 1 -o /tmp/fin $B > gpurun_out/proffin/ncu.log 2>&1
python tools/ncu_summary.py /tmp/fin.ncu-rep > gpurun_out/proffin/finalize_cfg1.summary.txt 2>&1
python tools/ncu_stalls.py /tmp/fin.ncu-rep 40 > gpurun_out/proffin/finalize_cfg1.stalls.txt 2>&1
python tools/ncu_lines.py /tmp/fin.ncu-rep 40 > gpurun_out/proffin/finalize_cfg1.lines.txt 2>&1 || true
cat gpurun_out/proffin/finalize_cfg1.summary.txt; head -45 gpurun_out/proffin/finalize_cfg1.stalls.txt
