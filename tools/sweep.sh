#!/bin/bash
# BASELINE config 4: throughput sweep over K x T x system x noise mode on one GPU; one bench.py
# JSON line per point into gpurun_out/sweep/, collated by tools/sweep_collate.py.  GPU box only.
#   K in 2^10, 2^14, 2^18, 2^22, 2^24; T in 50, 100, 200, 500; cartpole (cfg0 shape) and
#   quadrotor (cfg2 shape); Philox (noise in registers) and HBM (fp32 eps + jump tensors, drawn
#   on the device by the noise kernel).
# K*T cap: the HBM-mode tensors are 8 B (cartpole) / 28 B (quadrotor) per state-step, so the
# quadrotor at K = 2^24, T = 500 (235 GB) does not fit the 180 GB of HBM and is skipped; every
# other cell runs.
o=gpurun_out/sweep; mkdir -p $o
for noise in philox hbm; do
  for sys in cfg0 cfg2; do
    for t in 50 100 200 500; do
      for k in 1024 16384 262144 4194304 16777216; do
        if [ $noise = hbm ] && [ $sys = cfg2 ] && [ $k -eq 16777216 ] && [ $t -eq 500 ]; then continue; fi
        f=$o/${sys}_${noise}_K${k}_T${t}
        timeout 400 python bench.py --workload $sys --samples $k --horizon $t --noise $noise --steps 5 --warmup 3 \
          --no-cpu-baseline --no-e2e > $f.json 2> $f.err
      done
    done
  done
done
python tools/sweep_collate.py $o > $o/sweep_cfg4.md
