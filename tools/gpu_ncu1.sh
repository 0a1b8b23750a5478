#!/bin/bash
mkdir -p gpurun_out
SIGE_TC_TIMELINE=1 timeout 300 python tools/profile_layers.py --math tf32 --no-graphs > gpurun_out/timeline_tf32.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_conv_tc -s 322 -c 2 \
   -o gpurun_out/prof_v4 python tools/profile_layers.py --math tf32 --no-graphs > gpurun_out/ncu_v4.log 2>&1
exit 0
