#!/bin/bash
# Interleaved A/B of library variants (tools/bin/lib_<v>.so) vs the current build: tools/ab_bench.py.
mkdir -p gpurun_out
: > gpurun_out/ab_variants.txt
for r in 1 2 3; do
  timeout 200 python tools/ab_bench.py cur >> gpurun_out/ab_variants.txt 2>&1
  for v in "$@"; do
    SIGE_B200_LIB=tools/bin/lib_$v.so timeout 200 python tools/ab_bench.py $v >> gpurun_out/ab_variants.txt 2>&1
  done
done
exit 0
