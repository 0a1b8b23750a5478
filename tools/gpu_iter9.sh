#!/bin/bash
mkdir -p gpurun_out
: > gpurun_out/ab9.txt
for r in 1 2 3; do
  timeout 200 python tools/ab_bench.py cur >> gpurun_out/ab9.txt 2>&1
  SIGE_B200_LIB=tools/bin/lib_2981117.so timeout 200 python tools/ab_bench.py r1 >> gpurun_out/ab9.txt 2>&1
done
SIGE_B200_LIB=tools/bin/lib_marks.so SIGE_TC_GTL=1 timeout 300 python tools/graph_timeline.py > gpurun_out/tl_ph9.txt 2>gpurun_out/tl_ph9.err
timeout 900 python tools/grouped_probe.py 8 > gpurun_out/grouped_probe.txt 2>&1
timeout 1500 python -m pytest tests/test_gpu_engine.py tests/test_gpu_sharding.py tests/test_gpu_grouped.py tests/test_gpu_ops.py tests/test_gpu_expf.py -m gpu -q > gpurun_out/pytest_it9.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_it9.log
timeout 900 python bench.py > gpurun_out/bench_it9.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_it9.log
exit 0
