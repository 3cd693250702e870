#!/bin/bash
cd "$(dirname "$0")/.."
REGIONS="${REGIONS:-2x2 4x2 4x4}" python tools/cull_probe.py
for f in build/variants/*.so; do echo "== $f"; REGIONS="${REGIONS:-2x2 4x2 4x4}" RFB_LIB=$f python tools/cull_probe.py; done
