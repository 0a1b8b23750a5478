#!/bin/bash
# A/B of SIGE_TC_DEBUG experiment bits on the config-2 edit (interleaved, 3 rounds).
mkdir -p gpurun_out
out=gpurun_out/ab_dbg.txt
: > $out
for r in 1 2 3; do
  for d in "$@"; do
    SIGE_TC_DEBUG=$d timeout 300 python tools/ab_bench.py dbg$d >> $out 2>&1
  done
done
cat $out
