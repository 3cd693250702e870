#!/bin/bash
# Forward / train sweep over the view-culling region grid (RFB_VIEW_REGIONS)
cd "$(dirname "$0")/.."
for r in ${REGIONS:-1x1 2x2 4x2 4x4 8x4}; do
  echo "== RFB_VIEW_REGIONS=$r"
  RFB_VIEW_REGIONS=$r python tools/sweep_fwd.py --lanes 1 --cull 1 ${SWEEP_TRAIN---train} "$@"
done
