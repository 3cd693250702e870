#!/bin/bash
# A/B of the training step, default library vs variants, repeated (config 3 view, and the
# 3M surface scene's first orbit view)
cd "$(dirname "$0")/.."
for rep in 1 2; do
  python tools/sweep_fwd.py --lanes 1 --cull 1 --reps 10 --train 2>&1 | grep train | sed "s/^/default /"
  for f in build/variants/*.so; do RFB_LIB=$f python tools/sweep_fwd.py --lanes 1 --cull 1 --reps 10 --train 2>&1 | grep train | sed "s|^|$(basename $f) |"; done
done
