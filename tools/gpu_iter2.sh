#!/bin/bash
# Quick iteration: TC + engine parity, bench, per-CTA phase timeline.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_tc.py tests/test_gpu_engine.py -x -q > gpurun_out/pytest_it.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_it.log
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --requests 1 > gpurun_out/bench.log 2>&1
SIGE_TC_TIMELINE=1 timeout 300 python tools/profile_layers.py --math f16 --no-graphs > gpurun_out/cta_tl.log 2>&1
exit 0
