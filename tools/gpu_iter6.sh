#!/bin/bash
mkdir -p gpurun_out
SIGE_TC_GTL=1 timeout 300 python tools/graph_timeline.py > gpurun_out/tl_ph.txt 2>gpurun_out/tl_ph.err
timeout 900 python -m pytest tests/test_adapter.py tests/test_gpu_engine.py -m gpu -q -x -s > gpurun_out/pytest_ad.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_ad.log
exit 0
