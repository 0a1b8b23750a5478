#!/bin/bash
# Per-layer conv times of the config-2 edit under forced split plans (graph timeline, marks build).
mkdir -p gpurun_out
for plan in none 32:8:1 64:8:1 16:8:1 64:4:1 32:4:1; do
  if [ "$plan" = none ]; then
    SIGE_B200_LIB=tools/bin/lib_marks.so timeout 300 python tools/graph_timeline.py > gpurun_out/gs_$plan.txt 2>/dev/null
  else
    SIGE_FORCE_PLAN=$plan SIGE_B200_LIB=tools/bin/lib_marks.so timeout 300 python tools/graph_timeline.py > gpurun_out/gs_${plan//:/_}.txt 2>/dev/null
  fi
done
exit 0
