#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_config2.py tests/test_gpu_expf.py tests/test_gpu_engine.py -m gpu -q -s -x > gpurun_out/pytest_new.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_new.log
exit 0
