#!/bin/bash
mkdir -p gpurun_out
for M in tf32 f16; do
SIGE_TC_TIMELINE=1 timeout 300 python tools/profile_layers.py --math $M --no-graphs > gpurun_out/timeline_$M.log 2>&1
timeout 300 python tools/profile_layers.py --math $M > gpurun_out/layers_$M.log 2>&1
done
exit 0
