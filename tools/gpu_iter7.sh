#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_grouped.py tests/test_gpu_tc.py tests/test_gpu_engine.py -m gpu -q -x > gpurun_out/pytest_gr.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gr.log
timeout 600 python bench.py --requests 1 --no-cpu-baseline > gpurun_out/bench_it7.log 2>&1
SIGE_TC_GTL=1 timeout 300 python tools/graph_timeline.py > gpurun_out/tl_ph7.txt 2>gpurun_out/tl_ph7.err
exit 0
