#!/bin/bash
# ncu per-launch DRAM traffic / tensor-pipe activity of one bench.py sparse step (see tools/conv_traffic.py).
mkdir -p gpurun_out
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active \
  --clock-control none -c 2000 --csv --log-file gpurun_out/traffic.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline --requests 1 > gpurun_out/traffic_bench.log 2>&1
exit 0
