#!/bin/bash
# Source-level ncu of 4 sparse 256^2 conv launches (first sparse call, layers 1-4) + export pages.
mkdir -p gpurun_out
SIGE_NO_TUNE=1 timeout 900 ncu --set full --import-source on --clock-control none --cache-control none -k regex:k_conv_tc \
  --launch-skip 81 --launch-count 4 -f -o gpurun_out/prof_epi python tools/profile_layers.py --math f16 --no-graphs \
  > gpurun_out/ncu_epi.log 2>&1
for i in 0 1 2 3; do
  ncu -i gpurun_out/prof_epi.ncu-rep --page source --csv --print-source sass --launch-skip $i --launch-count 1 > gpurun_out/epi_src_$i.csv 2>/dev/null
done
ncu -i gpurun_out/prof_epi.ncu-rep --page details --csv > gpurun_out/epi_details.csv 2>/dev/null
exit 0
