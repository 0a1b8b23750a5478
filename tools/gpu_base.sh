#!/bin/bash
# Baseline pass: gpu tests, smoke, bench (repo arm), graph timeline.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
SIGE_TC_GTL=1 timeout 300 python tools/graph_timeline.py > gpurun_out/tl.txt 2>gpurun_out/tl.err
exit 0
