#!/bin/bash
# round-2 state check on the GPU box: gpu tests, bench lines of every workload, launch list.
o=gpurun_out/state; mkdir -p $o
python -m pytest tests -m gpu -x -q > $o/pytest_gpu.txt 2>&1; echo "pytest exit $?" >> $o/pytest_gpu.txt
python bench.py > $o/bench_cfg1.json 2> $o/bench_cfg1.err
python bench.py --impl reference --steps 3 --warmup 1 > $o/bench_ref.json 2> $o/bench_ref.err
for wl in cfg0 cfg2 cfg3; do
  python bench.py --workload $wl --no-cpu-baseline > $o/bench_$wl.json 2> $o/bench_$wl.err
done
python bench.py --workload cfg1 --noise hbm --samples 1048576 --no-cpu-baseline --no-e2e > $o/bench_hbm_cart1M.json 2> $o/bench_hbm_cart1M.err
python bench.py --workload cfg3 --noise hbm --no-cpu-baseline --no-e2e > $o/bench_hbm_cfg3.json 2> $o/bench_hbm_cfg3.err
python bench.py --workload cfg1 --samples 1048576 --no-cpu-baseline --no-e2e > $o/bench_cart1M.json 2> $o/bench_cart1M.err
python bench.py --precision f64 --no-cpu-baseline > $o/bench_cfg1_f64.json 2> $o/bench_cfg1_f64.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $o/launches_cfg1.csv python bench.py --steps 2 --warmup 1 --profile --no-cpu-baseline --no-e2e > $o/ncu_launch.log 2>&1
