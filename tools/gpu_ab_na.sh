#!/bin/bash
# A/B of the static-launch A-ring sizing (SIGE_NA_FULL=1 restores kMaxNA slots).
mkdir -p gpurun_out
for i in 1 2; do
timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --requests 1 > gpurun_out/ab_new_$i.log 2>&1
SIGE_NA_FULL=1 timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --requests 1 > gpurun_out/ab_old_$i.log 2>&1
done
exit 0
