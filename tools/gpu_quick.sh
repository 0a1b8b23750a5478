#!/bin/bash
# GPU tests (tensor-core + engine + ops) and two short benches.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pt.log 2>&1
for i in 1 2; do
timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --requests 1 > gpurun_out/q_$i.log 2>&1
done
exit 0
