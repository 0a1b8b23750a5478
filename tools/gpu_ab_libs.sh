#!/bin/bash
# A/B of library builds on the config-2 edit (interleaved rounds): cur vs tools/bin/lib_<name>.so
mkdir -p gpurun_out
out=gpurun_out/ab_libs.txt
: > $out
for r in 1 2 3 4; do
  timeout 300 python tools/ab_bench.py cur >> $out 2>&1
  for n in "$@"; do
    SIGE_B200_LIB=tools/bin/lib_$n.so timeout 300 python tools/ab_bench.py $n >> $out 2>&1
  done
done
cat $out
