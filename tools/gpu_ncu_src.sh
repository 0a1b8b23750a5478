#!/bin/bash
# Source-level ncu capture of a few conv launches inside one sparse edit (no graphs, no tuner trials;
# caches NOT flushed between replays, so the profile resembles the warm steady state).
# usage: bash tools/gpu_ncu_src.sh SKIP COUNT
mkdir -p gpurun_out
SIGE_NO_TUNE=1 timeout 900 ncu --set full --import-source on --clock-control none --cache-control none -k regex:k_conv_tc \
  --launch-skip "$1" --launch-count "$2" -f -o gpurun_out/prof_src python tools/profile_layers.py --math f16 --no-graphs \
  > gpurun_out/ncu_src.log 2>&1
exit 0
