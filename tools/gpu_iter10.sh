#!/bin/bash
mkdir -p gpurun_out
: > gpurun_out/ab10.txt
for r in 1 2 3; do
  timeout 200 python tools/ab_bench.py handoff >> gpurun_out/ab10.txt 2>&1
  SIGE_NO_CTR_HANDOFF=1 timeout 200 python tools/ab_bench.py pdl >> gpurun_out/ab10.txt 2>&1
done
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_it10.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_it10.log
SIGE_B200_LIB=tools/bin/lib_marks.so SIGE_TC_GTL=1 timeout 300 python tools/graph_timeline.py > gpurun_out/tl_ph10.txt 2>gpurun_out/tl_ph10.err
exit 0
