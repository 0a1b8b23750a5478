#!/bin/bash
mkdir -p gpurun_out
for D in 0; do
SIGE_TC_DEBUG=$D SIGE_TC_TIMELINE=1 timeout 300 python tools/profile_layers.py --math tf32 --no-graphs > gpurun_out/timeline_dbg$D.log 2>&1
done
for M in tf32 f16; do timeout 300 python tools/profile_layers.py --math $M > gpurun_out/layers_$M.log 2>&1; done
timeout 900 python -m pytest tests/test_gpu_tc.py -x -q > gpurun_out/pytest_tc.log 2>&1
exit 0
