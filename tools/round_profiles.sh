#!/bin/bash
# Bench lines for every config + the launch list of the default bench (profiles/)
cd "$(dirname "$0")/.."
T=${TAG:-r2l}
python bench.py --config 4 > gpurun_out/${T}_bench_config4.json 2> gpurun_out/${T}_bench_config4.err
python bench.py --config 5 --steps 5 > gpurun_out/${T}_bench_config5.json 2> gpurun_out/${T}_bench_config5.err
python bench.py --quantile --no-train-iter --no-adjacency > gpurun_out/${T}_bench_quantile.json 2> gpurun_out/${T}_bench_quantile.err
python bench.py --config 1 > gpurun_out/${T}_bench_config1.json 2> gpurun_out/${T}_bench_config1.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${T}_launches.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-parity --no-e2e --no-train-iter --no-adjacency > gpurun_out/${T}_ncu_launch.log 2>&1
