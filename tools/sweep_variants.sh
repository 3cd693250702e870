#!/bin/bash
# Run the forward/train sweep for the default library and every build/variants/*.so
cd "$(dirname "$0")/.."
python tools/sweep_fwd.py --lanes 1 ${SWEEP_TRAIN---train} "$@"
for f in $(ls build/variants/*.so 2>/dev/null); do RFB_LIB=$f python tools/sweep_fwd.py --lanes 1 ${SWEEP_TRAIN---train} "$@"; done
