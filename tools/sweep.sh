#!/bin/bash
# BASELINE config 4: throughput sweep over K x T x system (x noise mode), one JSON line per
# point into gpurun_out/sweep/<system>_<noise>_K<k>_T<t>.json.  GPU box only.
o=gpurun_out/sweep; mkdir -p $o
for sys in cfg0 cfg2; do            # cartpole / quadrotor single iterations at the swept shape
  for t in 50 100 200 500; do
    for k in 1024 16384 262144 4194304 16777216; do
      if [ $sys = cfg2 ] && [ $k -gt 4194304 ] && [ $t -gt 200 ]; then continue; fi
      timeout 240 python bench.py --workload $sys --samples $k --horizon $t --steps 5 --warmup 3 \
        --no-cpu-baseline --no-e2e > $o/${sys}_philox_K${k}_T${t}.json 2> $o/${sys}_philox_K${k}_T${t}.err
    done
  done
  for t in 100 200; do
    for k in 262144 1048576 4194304; do
      timeout 240 python bench.py --workload $sys --samples $k --horizon $t --noise hbm --steps 5 --warmup 3 \
        --no-cpu-baseline --no-e2e > $o/${sys}_hbm_K${k}_T${t}.json 2> $o/${sys}_hbm_K${k}_T${t}.err
    done
  done
done
