#!/bin/bash
o=gpurun_out/b7; mkdir -p $o
python -m pytest tests -m gpu -x -q > $o/pytest_gpu.txt 2>&1; echo "pytest exit $?" >> $o/pytest_gpu.txt
tail -3 $o/pytest_gpu.txt
for a in "--workload cfg1 --noise hbm --samples 1048576" "--workload cfg3 --noise hbm" "--workload cfg1" "--workload cfg3"; do echo "$a: $(python bench.py $a --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d[\"roofline\"]; print(round(d[\"ms_per_step\"]*1e3,2), round(r[\"kernel_ms\"]*1e3,2), (r.get(\"hbm\") or {}).get(\"frac\"))")"; done | tee $o/ab.txt
