#!/bin/bash
# Iteration pass: targeted tests, bench (no cpu baseline), graph timeline with plans.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_splitk.py tests/test_gpu_engine.py tests/test_gpu_tc.py -m gpu -q -x -s > gpurun_out/pytest_it.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_it.log
timeout 600 python bench.py --no-cpu-baseline --requests 1 > gpurun_out/bench_it.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_it.log
SIGE_TC_GTL=1 timeout 300 python tools/graph_timeline.py > gpurun_out/tl_it.txt 2>gpurun_out/tl_it.err
exit 0
