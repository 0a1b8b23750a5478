#!/bin/bash
mkdir -p gpurun_out
timeout 600 python bench.py --requests 1 --no-cpu-baseline > gpurun_out/bench_pf.log 2>&1
SIGE_NO_L2_PREFETCH=1 timeout 600 python bench.py --requests 1 --no-cpu-baseline > gpurun_out/bench_nopf.log 2>&1
timeout 600 python bench.py --requests 1 --no-cpu-baseline > gpurun_out/bench_pf2.log 2>&1
SIGE_TC_GTL=1 timeout 300 python tools/graph_timeline.py > gpurun_out/tl_pf.txt 2>gpurun_out/tl_pf.err
SIGE_TC_TIMELINE=1 timeout 300 python tools/profile_layers.py --math f16 --no-graphs > gpurun_out/cta_tl.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_engine.py tests/test_gpu_ops.py tests/test_gpu_splitk.py tests/test_gpu_config2.py -m gpu -q -x > gpurun_out/pytest_it.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_it.log
exit 0
