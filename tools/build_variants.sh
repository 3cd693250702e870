#!/bin/bash
# Build librfb.so variants (compile-time knobs) into build/variants/ for sweeps.
set -e
cd "$(dirname "$0")/.."
mkdir -p build/variants
for spec in "$@"; do
  name=$(echo "$spec" | tr ' =' '_-')
  flags=""
  for kv in $spec; do flags="$flags -D$kv"; done
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -fmad=false -std=c++17 $flags \
       -Xcompiler -fPIC -shared -o build/variants/librfb_$name.so paper_2502_01157_b200/csrc/rfb.cu \
       paper_2502_01157_b200/csrc/rfb_adjacency.cu paper_2502_01157_b200/csrc/rfb_segments.cu &
done
wait
ls build/variants
