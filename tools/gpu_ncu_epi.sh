#!/bin/bash
# Source-level ncu of 2 sparse 256^2 conv launches (first sparse call, layers 1-2); report in /tmp, CSV pages back.
mkdir -p gpurun_out
SIGE_NO_TUNE=1 timeout 900 ncu --set full --import-source on --clock-control none --cache-control none -k regex:k_conv_tc \
  --launch-skip 81 --launch-count 2 -f -o /tmp/prof_epi python tools/profile_layers.py --math f16 --no-graphs \
  > gpurun_out/ncu_epi.log 2>&1
for i in 0 1; do
  ncu -i /tmp/prof_epi.ncu-rep --page source --csv --print-source sass --launch-skip $i --launch-count 1 > /tmp/epi_src_$i.csv 2>/dev/null
  python tools/sass_hot.py /tmp/epi_src_$i.csv 80 > gpurun_out/epi_hot_$i.txt 2>&1
done
ncu -i /tmp/prof_epi.ncu-rep --page details --csv > gpurun_out/epi_details.csv 2>/dev/null
ls -la /tmp/prof_epi.ncu-rep /tmp/epi_src_*.csv >> gpurun_out/ncu_epi.log
exit 0
