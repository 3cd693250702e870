#!/bin/bash
cd "$(dirname "$0")/.."
python tools/sweep_fwd.py --lanes 1 --cull 1 --train > gpurun_out/r3m_split.txt 2>&1
RFB_LIB=build/variants/librfb_RFB_NO_REVERSE.so python tools/sweep_fwd.py --lanes 1 --cull 1 --train >> gpurun_out/r3m_split.txt 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_train -c 1 -o gpurun_out/r3m_prof_train python tools/sweep_fwd.py --lanes 1 --cull 1 --once --train > gpurun_out/r3m_ncu_train.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_render -c 1 -o gpurun_out/r3m_prof_render python tools/sweep_fwd.py --lanes 1 --cull 1 --once > gpurun_out/r3m_ncu_render.log 2>&1
