#!/bin/bash
mkdir -p gpurun_out
SIGE_TC_TIMELINE=1 timeout 300 python tools/profile_layers.py --math tf32 --no-graphs > gpurun_out/timeline_tf32.log 2>&1
exit 0
