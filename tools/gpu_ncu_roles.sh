#!/bin/bash
# ncu stall sampling of conv launches per warp role (tools/ncu_roles.py):
# launches SKIP..SKIP+COUNT-1 of tools/profile_layers.py (80 = first sparse edit's layer 0).
# usage: bash tools/gpu_ncu_roles.sh SKIP COUNT TAG
mkdir -p gpurun_out
SIGE_NO_TUNE=1 timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_conv_tc \
  --launch-skip "$1" --launch-count "$2" -f -o /tmp/prof_roles python tools/profile_layers.py --math f16 --no-graphs \
  > gpurun_out/ncu_roles_$3.log 2>&1
cuobjdump -xelf all paper_2211_02048_b200/lib/libsige_b200.so > /dev/null 2>&1

nvdisasm -g conv_tc.sm_100a.cubin > /tmp/all.sass 2>/dev/null
rm -f *.cubin
for i in $(seq 0 $(($2 - 1))); do
  ncu -i /tmp/prof_roles.ncu-rep --page source --csv --print-source sass --launch-skip $i --launch-count 1 > /tmp/roles_$i.csv 2>/dev/null
  k=$(ncu -i /tmp/prof_roles.ncu-rep --page raw --csv --launch-skip $i --launch-count 1 2>/dev/null | sed -n 3p | cut -d, -f5 | tr -d '"' | sed 's/<.*//')
  echo "== launch $(($1 + i)) $(ncu -i /tmp/prof_roles.ncu-rep --page raw --csv --launch-skip $i --launch-count 1 --metrics gpu__time_duration.sum 2>/dev/null | tail -1 | awk -F'","' '{print $NF}')" >> gpurun_out/ncu_roles_$3.txt
  python tools/ncu_roles.py /tmp/roles_$i.csv /tmp/all.sass "k_conv_tcILb1ELi3ELi1ELb0E" 45 | grep -v " 0   0.0%" >> gpurun_out/ncu_roles_$3.txt 2>&1
done
exit 0
