# one ncu --set full capture of the rollout kernel: tools/prof1.sh <name> <env> <bench args...>
set -e
name=$1; shift; envs=$1; shift
B="python bench.py --steps 2 --warmup 1 --profile --no-cpu-baseline --no-e2e $*"
env $envs $B > gpurun_out/plain_$name.log 2>&1
env $envs ncu --set full --clock-control none --import-source on -k regex:rollout_ -s 2 -c 1 -o /tmp/prof_$name $B > gpurun_out/ncu_$name.log 2>&1
python tools/ncu_summary.py /tmp/prof_$name.ncu-rep > gpurun_out/prof_$name.summary.txt 2>&1
python tools/ncu_stalls.py /tmp/prof_$name.ncu-rep 60 > gpurun_out/prof_$name.stalls.txt 2>&1
ncu -i /tmp/prof_$name.ncu-rep --page raw --csv > gpurun_out/prof_$name.raw.csv 2>&1
python tools/ncu_lines.py /tmp/prof_$name.ncu-rep 70 > gpurun_out/prof_$name.lines.txt 2>&1 || true
