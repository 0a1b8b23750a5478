#!/bin/bash
# Quick iteration: GPU tests (tensor-core + engine), per-layer timing in both TC modes.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for M in tf32 f16; do
timeout 300 python tools/profile_layers.py --math $M > gpurun_out/layers_$M.log 2>&1
done
SIGE_TC_TIMELINE=1 timeout 300 python tools/profile_layers.py --math tf32 --no-graphs > gpurun_out/timeline_tf32.log 2>&1
exit 0
