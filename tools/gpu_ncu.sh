#!/bin/bash
# ncu --set full of one kernel on the C5 element type (small mesh). usage: bash tools/gpu_ncu.sh TAG REGEX
TAG=${1:-n}; RX=${2:-rhs2_kernel}
mkdir -p gpurun_out
timeout 300 python tools/profile_run.py 3 12 8 2 > gpurun_out/${TAG}_prof_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$RX" -s 1 -c 1 \
  -o gpurun_out/${TAG}_prof python tools/profile_run.py 3 12 8 2 > gpurun_out/${TAG}_ncu_full.log 2>&1
echo "ncu rc=$?"
