#!/bin/bash
# Per-CTA phase marks of every conv launch (non-graph run; see SIGE_TC_TIMELINE in conv_tc.cu).
# usage: bash tools/gpu_cta_tl.sh [SIGE_TC_DEBUG values to compare...]
mkdir -p gpurun_out
SIGE_TC_TIMELINE=1 timeout 300 python tools/profile_layers.py --math f16 --no-graphs > gpurun_out/cta_tl.log 2>&1
for d in "$@"; do
  SIGE_TC_DEBUG=$d SIGE_TC_TIMELINE=1 timeout 300 python tools/profile_layers.py --math f16 --no-graphs > gpurun_out/cta_tl_d$d.log 2>&1
done
exit 0
