#!/bin/bash
mkdir -p gpurun_out
SIGE_TC_TIMELINE=1 timeout 300 python tools/profile_layers.py --math f16 --no-graphs > gpurun_out/timeline_f16.log 2>&1
SIGE_NO_PDL=1 SIGE_TC_TIMELINE=1 timeout 300 python tools/profile_layers.py --math f16 --no-graphs > gpurun_out/timeline_f16_nopdl.log 2>&1
timeout 300 python tools/profile_layers.py --math f16 > gpurun_out/layers_f16.log 2>&1
SIGE_NO_PDL=1 timeout 300 python tools/profile_layers.py --math f16 > gpurun_out/layers_f16_nopdl.log 2>&1
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_pdl.log 2>&1
SIGE_NO_PDL=1 timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_nopdl.log 2>&1
exit 0
