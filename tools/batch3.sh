#!/bin/bash
# A/B batch 3: main (quadrotor SFU sincos + grouped cost + diagonal Cholesky form) vs v3 (cartpole SFU sincos)
o=gpurun_out/b3; mkdir -p $o
JM_GATE_REPORT=$o/gate_main.jsonl python -m pytest tests -m gpu -x -q > $o/pytest_gpu.txt 2>&1; echo "pytest exit $?" >> $o/pytest_gpu.txt
JM_LIB=scratch/libjm_v3.so JM_GATE_REPORT=$o/gate_v3.jsonl python -m pytest tests/test_gpu_f32_gate.py tests/test_gpu_parity.py -q > $o/pytest_v3.txt 2>&1; echo "pytest exit $?" >> $o/pytest_v3.txt
export OUT=$o/ab.txt STEPS=10
EXTRA_WL="--workload cfg3 --noise hbm" bash tools/ab.sh "JM_X=0" "JM_LIB=scratch/libjm_v3.so"
for wl in cfg2 cfg0 "cfg1 --samples 1048576"; do
  for envs in "JM_X=0" "JM_LIB=scratch/libjm_v3.so"; do
    echo "$wl $envs $(env $envs python bench.py --workload $wl --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"]*1e3, d["roofline"]["kernel_ms"]*1e3, d["roofline"]["kernel"])')" >> $o/ab.txt
  done
done
cat $o/ab.txt
