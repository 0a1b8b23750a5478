#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_ops.py -m gpu -q -x > gpurun_out/pytest_it11.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_it11.log
timeout 300 python tools/ops_hbm.py > gpurun_out/ops_hbm_tma.txt 2>&1
SIGE_NO_TMA_GATHER=1 timeout 300 python tools/ops_hbm.py > gpurun_out/ops_hbm_notma.txt 2>&1
exit 0
