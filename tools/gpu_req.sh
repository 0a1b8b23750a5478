#!/bin/bash
mkdir -p gpurun_out
timeout 900 python tools/requests.py > gpurun_out/requests.jsonl 2> gpurun_out/requests.err
exit 0
