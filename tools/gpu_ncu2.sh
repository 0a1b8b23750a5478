#!/bin/bash
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_conv_tc -s 321 -c 1 \
   -o gpurun_out/prof_act python tools/profile_layers.py --math tf32 --no-graphs > gpurun_out/ncu_act.log 2>&1
exit 0
