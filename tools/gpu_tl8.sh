#!/bin/bash
mkdir -p gpurun_out
SIGE_TC_TIMELINE=1 timeout 300 python tools/profile_layers.py --math f16 --no-graphs > gpurun_out/timeline_f16.log 2>&1
exit 0
