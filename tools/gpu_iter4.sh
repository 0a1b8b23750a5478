#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_splitk.py tests/test_gpu_engine.py tests/test_gpu_ops.py tests/test_gpu_expf.py -m gpu -q -x > gpurun_out/pytest_it.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_it.log
timeout 600 python bench.py --requests 1 > gpurun_out/bench_it.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_it.log
SIGE_TC_TIMELINE=1 timeout 300 python tools/profile_layers.py --math f16 --no-graphs > gpurun_out/cta_tl.log 2>&1
exit 0
