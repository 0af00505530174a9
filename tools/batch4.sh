#!/bin/bash
# A/B batch 4: CTA size of the packed (two samples per thread) kernels: 256 (main) / 288 / 320 threads
o=gpurun_out/b4; mkdir -p $o
python -m pytest tests -m gpu -x -q > $o/pytest_gpu.txt 2>&1; echo "pytest exit $?" >> $o/pytest_gpu.txt
export OUT=$o/ab.txt STEPS=10
EXTRA_WL="--workload cfg3 --noise hbm" bash tools/ab.sh "JM_X=0" "JM_LIB=scratch/libjm_p288.so" "JM_LIB=scratch/libjm_p320.so"
for envs in "JM_X=0" "JM_LIB=scratch/libjm_p288.so" "JM_LIB=scratch/libjm_p320.so"; do
  echo "cart1M $envs $(env $envs python bench.py --workload cfg1 --samples 1048576 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"]*1e3, d["roofline"]["kernel_ms"]*1e3, d["roofline"]["kernel"])')" >> $o/ab.txt
done
cat $o/ab.txt
