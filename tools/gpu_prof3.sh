#!/bin/bash
# Config-4 sweep, launch list, per-launch DRAM bytes of one sparse step's convs, ncu --set full of two convs.
mkdir -p gpurun_out
timeout 600 python tools/sweep.py > gpurun_out/sweep.jsonl 2> gpurun_out/sweep.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 1400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_ncu.log 2>&1
# bench: precompute 80 convs (+ tuning trials) ... skip to the timed step's convs: use -k and a large skip computed from the launch list offline
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:k_conv_tc --csv --log-file gpurun_out/conv_dram.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/bench_ncu2.log 2>&1
exit 0
