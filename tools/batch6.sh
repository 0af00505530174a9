#!/bin/bash
o=gpurun_out/b6; mkdir -p $o
python -m pytest tests -m gpu -x -q > $o/pytest_gpu.txt 2>&1; echo "pytest exit $?" >> $o/pytest_gpu.txt
tail -5 $o/pytest_gpu.txt
for a in "--workload cfg1" "--workload cfg3" "--workload cfg1 --samples 1048576" "--workload cfg2" "--workload cfg0" "--workload cfg1 --nu 0" "--workload cfg3 --nu 0"; do echo "$a: $(python bench.py $a --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d[\"ms_per_step\"]*1e3,2), round(d[\"roofline\"][\"kernel_ms\"]*1e3,2))")"; done | tee $o/ab.txt
