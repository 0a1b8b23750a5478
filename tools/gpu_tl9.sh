#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_ops.py -x -q > gpurun_out/pytest_ops.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_ops.log
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench.log 2>&1
exit 0
