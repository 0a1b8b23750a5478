#!/bin/bash
# Tests + per-layer timing + one ncu --set full capture of k_conv_tc launches.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python tools/profile_layers.py > gpurun_out/layers.log 2>&1
SIGE_TC_TIMELINE=1 timeout 300 python tools/profile_layers.py --no-graphs > gpurun_out/timeline.log 2>&1
# sparse step launches: skip precompute/warmup kernels, capture a few convs of the sparse step
for S in 330 365; do
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_conv_tc -s $S -c 3 \
   -o gpurun_out/prof_conv_$S python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full_$S.log 2>&1
done
exit 0
