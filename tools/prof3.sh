set -e
make -j16 >/dev/null 2>&1
B="python bench.py --steps 2 --warmup 1 --profile --no-cpu-baseline --no-e2e"
JM_SPT=1 $B --workload cfg3 > gpurun_out/plain.log 2>&1
JM_SPT=1 ncu --set full --clock-control none --import-source on -k regex:rollout_fast -s 2 -c 1 -o gpurun_out/prof_cfg3_spt1 $B --workload cfg3 > gpurun_out/ncu1.log 2>&1
JM_SPT=2 $B --workload cfg3 > gpurun_out/plain.log 2>&1
JM_SPT=2 ncu --set full --clock-control none --import-source on -k regex:rollout_fast -s 2 -c 1 -o gpurun_out/prof_cfg3_spt2 $B --workload cfg3 > gpurun_out/ncu2.log 2>&1
JM_SPT=1 $B --workload cfg1 > gpurun_out/plain.log 2>&1
JM_SPT=1 ncu --set full --clock-control none --import-source on -k regex:rollout_fast -s 2 -c 1 -o gpurun_out/prof_cfg1_spt1 $B --workload cfg1 > gpurun_out/ncu3.log 2>&1
ls -la gpurun_out/*.ncu-rep
for r in gpurun_out/prof_*.ncu-rep; do
  python tools/ncu_summary.py $r > ${r%.ncu-rep}.summary.txt 2>&1
  python tools/ncu_stalls.py $r 40 > ${r%.ncu-rep}.stalls.txt 2>&1
  ncu -i $r --page raw --csv > ${r%.ncu-rep}.raw.csv 2>&1
done
mkdir -p /tmp/reps && mv gpurun_out/prof_*.ncu-rep /tmp/reps/
