#!/bin/bash
# Graph timeline of the config-2 edit under forced static plans (SIGE_FORCE_PLAN=nt:ks).
mkdir -p gpurun_out
for P in none 32:8 64:8 16:4 16:8 32:4 128:8; do
  if [ "$P" = none ]; then unset SIGE_FORCE_PLAN; else export SIGE_FORCE_PLAN=$P; fi
  SIGE_TC_GTL=1 timeout 300 python tools/graph_timeline.py > gpurun_out/tlp_${P/:/_}.txt 2>gpurun_out/tlp_${P/:/_}.err
done
unset SIGE_FORCE_PLAN
timeout 1200 python -m pytest tests/test_gpu_splitk.py tests/test_gpu_engine.py -m gpu -q -x -s > gpurun_out/pytest_it.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_it.log
exit 0
