#!/bin/bash
# A/B one environment switch: TC + engine parity suites (default build), then bench + graph timeline
# with and without the switch.   usage: bash tools/gpu_ab.sh VAR=value
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_tc.py tests/test_gpu_engine.py -x -q > gpurun_out/pytest_ab.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_ab.log
for r in 1 2; do
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --requests 1 > gpurun_out/bench_a$r.log 2>&1
env "$1" timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --requests 1 > gpurun_out/bench_b$r.log 2>&1
done
SIGE_TC_GTL=1 timeout 300 python tools/graph_timeline.py > gpurun_out/tl_a.log 2>&1
env "$1" SIGE_TC_GTL=1 timeout 300 python tools/graph_timeline.py > gpurun_out/tl_b.log 2>&1
exit 0
