#!/bin/bash
# One ncu --set full capture of two config-2 conv launches (a sparse 256^2 layer and an 8x8 dense-fallback
# layer of the first sparse edit), summarised into gpurun_out/ncu_full_summary.txt.
mkdir -p gpurun_out
SIGE_NO_TUNE=1 timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_conv_tc \
  --launch-skip 81 --launch-count 1 -f -o /tmp/full_sparse python tools/profile_layers.py --math f16 --no-graphs \
  > gpurun_out/ncu_full.log 2>&1
SIGE_NO_TUNE=1 timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_conv_tc \
  --launch-skip 108 --launch-count 1 -f -o /tmp/full_fb python tools/profile_layers.py --math f16 --no-graphs \
  >> gpurun_out/ncu_full.log 2>&1
for r in sparse fb; do
  echo "== $r" >> gpurun_out/ncu_full_summary.txt
  ncu -i /tmp/full_$r.ncu-rep --page details --csv 2>/dev/null | python3 -c '
import csv, sys
keep = ("Duration", "Compute (SM) Throughput", "Memory Throughput", "DRAM Throughput", "L2 Cache Throughput",
        "Registers Per Thread", "Achieved Occupancy", "Executed Ipc Active", "Issue Slots Busy",
        "No Eligible", "Warp Cycles Per Issued Instruction", "Dynamic Shared Memory Per Block", "Grid Size",
        "L1/TEX Hit Rate", "L2 Hit Rate")
for r in csv.reader(sys.stdin):
    if len(r) > 14 and r[12] in keep:
        print(f"{r[11][:34]:34s} | {r[12]:36s} | {r[14]} {r[13]}")
' >> gpurun_out/ncu_full_summary.txt
  ncu -i /tmp/full_$r.ncu-rep --page raw --csv --metrics dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__inst_executed_pipe_uniform.sum 2>/dev/null | tail -2 >> gpurun_out/ncu_full_summary.txt
done
exit 0
