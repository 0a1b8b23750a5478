#!/bin/bash
# A/B of library builds from earlier commits (tools/bin/lib_<commit>.so) vs the current build, interleaved.
mkdir -p gpurun_out
: > gpurun_out/ab_commits.txt
for r in 1 2 3; do
  timeout 200 python tools/ab_bench.py cur >> gpurun_out/ab_commits.txt 2>&1
  for c in 2981117 97f121a 534fd0f; do
    SIGE_B200_LIB=tools/bin/lib_$c.so timeout 200 python tools/ab_bench.py $c >> gpurun_out/ab_commits.txt 2>&1
  done
done
exit 0
