#!/bin/bash
# A/B of an environment switch on the config-2 edit (interleaved rounds): bash tools/gpu_ab_env.sh VAR=VALUE
mkdir -p gpurun_out
out=gpurun_out/ab_env.txt
: > $out
for r in 1 2 3 4; do
  timeout 300 python tools/ab_bench.py base >> $out 2>&1
  env "$@" timeout 300 python tools/ab_bench.py "$*" >> $out 2>&1
done
cat $out
