#!/bin/bash
# Graph timeline of one config-2 edit (per-launch spans + the [gtl i] launch descriptions on stderr).
mkdir -p gpurun_out
SIGE_TC_GTL=1 timeout 300 python tools/graph_timeline.py > gpurun_out/tl.log 2> gpurun_out/tl_desc.log
exit 0
