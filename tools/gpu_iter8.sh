#!/bin/bash
mkdir -p gpurun_out
timeout 600 python bench.py --requests 1 --no-cpu-baseline > gpurun_out/bench_it8.log 2>&1
SIGE_B200_LIB=tools/bin/lib_marks.so SIGE_TC_GTL=1 timeout 300 python tools/graph_timeline.py > gpurun_out/tl_ph8.txt 2>gpurun_out/tl_ph8.err
timeout 900 python tools/grouped_probe.py 8 16 32 > gpurun_out/grouped_probe.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_engine.py tests/test_gpu_sharding.py -m gpu -q -x > gpurun_out/pytest_it8.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_it8.log
exit 0
