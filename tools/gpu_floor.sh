#!/bin/bash
mkdir -p gpurun_out
SIGE_TC_GTL=1 timeout 300 python tools/graph_timeline.py > gpurun_out/graph_timeline.log 2>&1
SIGE_TC_DEBUG=1024 SIGE_TC_GTL=1 timeout 300 python tools/graph_timeline.py > gpurun_out/graph_timeline_floor.log 2>&1
exit 0
