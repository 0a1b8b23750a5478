#!/bin/bash
# ncu (full set) of grouped-call conv launches (tools/grouped_profile.py R --no-graphs; launch 80 = first grouped
# call's layer 0): per-role stall breakdown + the details page. usage: bash tools/gpu_ncu_grouped.sh R SKIP COUNT
mkdir -p gpurun_out
SIGE_NO_TUNE=1 timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_conv_tc \
  --launch-skip "$2" --launch-count "$3" -f -o /tmp/prof_grp python tools/grouped_profile.py "$1" --no-graphs \
  > gpurun_out/ncu_grp.log 2>&1
cuobjdump -xelf all paper_2211_02048_b200/lib/libsige_b200.so > /dev/null 2>&1
nvdisasm -g conv_tc.sm_100a.cubin > /tmp/all.sass 2>/dev/null
rm -f *.cubin
for i in $(seq 0 $(($3 - 1))); do
  ncu -i /tmp/prof_grp.ncu-rep --page source --csv --print-source sass --launch-skip $i --launch-count 1 > /tmp/grp_$i.csv 2>/dev/null
  echo "== launch $(($2 + i))" >> gpurun_out/ncu_grp_roles.txt
  python tools/ncu_roles.py /tmp/grp_$i.csv /tmp/all.sass "k_conv_tcILb1ELi3ELi1ELb0E" 40 | grep -v " 0   0.0%" >> gpurun_out/ncu_grp_roles.txt 2>&1
done
ncu -i /tmp/prof_grp.ncu-rep --page details --csv > gpurun_out/ncu_grp_details.csv 2>/dev/null
exit 0
