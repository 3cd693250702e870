set -x
ncu --set full --clock-control none --import-source on -k regex:k_train -c 1 -o gpurun_out/r3c_prof_train python tools/sweep_fwd.py --lanes 1 --once --train > gpurun_out/r3c_ncu_train.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_render -c 1 -o gpurun_out/r3c_prof_render python tools/sweep_fwd.py --lanes 1 --once > gpurun_out/r3c_ncu_render.log 2>&1
