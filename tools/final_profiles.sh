#!/bin/bash
# Round-end artifacts at HEAD: bench lines for every config, ncu captures of the two hot
# kernels, the launch list of the default bench (profiles/, tag $TAG)
cd "$(dirname "$0")/.."
T=${TAG:-r2p}
python bench.py > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
python bench.py --config 4 > gpurun_out/${T}_bench_config4.json 2> gpurun_out/${T}_bench_config4.err
python bench.py --config 5 --steps 5 > gpurun_out/${T}_bench_config5.json 2> gpurun_out/${T}_bench_config5.err
python bench.py --quantile --no-train-iter --no-adjacency > gpurun_out/${T}_bench_quantile.json 2> gpurun_out/${T}_bench_quantile.err
python bench.py --config 1 > gpurun_out/${T}_bench_config1.json 2> gpurun_out/${T}_bench_config1.err
ncu --set full --clock-control none --import-source on -k regex:k_train -c 1 -o gpurun_out/${T}_prof_train python tools/sweep_fwd.py --lanes 1 --cull 1 --once --train > gpurun_out/${T}_ncu_train.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_render -c 1 -o gpurun_out/${T}_prof_render python tools/sweep_fwd.py --lanes 1 --cull 1 --once > gpurun_out/${T}_ncu_render.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${T}_launches.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-parity --no-e2e --no-train-iter --no-adjacency > gpurun_out/${T}_ncu_launch.log 2>&1
