#!/bin/bash
# ncu launch list (gpu__time_duration + DRAM bytes per launch) of a short default bench.py run; summary via launch_summary.py.
mkdir -p gpurun_out
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 2000 --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --sweep 0 --spade 0 --requests 1 --no-cpu-baseline \
  > gpurun_out/launches_bench.log 2>&1
python tools/launch_summary.py gpurun_out/launches.csv > gpurun_out/launches_summary.txt 2>&1
python tools/conv_traffic.py gpurun_out/launches.csv > gpurun_out/conv_traffic.txt 2>&1
exit 0
