#!/bin/bash
# A/B of two builds of the library (SIGE_B200_LIB override): $1 = alternative .so (relative path)
mkdir -p gpurun_out
for i in 1 2 3; do
timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --requests 1 > gpurun_out/ab_cur_$i.log 2>&1
SIGE_B200_LIB=$1 timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --requests 1 > gpurun_out/ab_alt_$i.log 2>&1
done
exit 0
