#!/bin/bash
# ncu --set full of K1 and K3 (one launch each) on the C5 element type. usage: bash tools/gpu_ncu2.sh TAG
TAG=${1:-n2}
mkdir -p gpurun_out
timeout 300 python tools/profile_run.py 3 12 8 2 > gpurun_out/${TAG}_prof_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"project_kernel|wadj3" -s 2 -c 2 \
  -o gpurun_out/${TAG}_k13 python tools/profile_run.py 3 12 8 2 > gpurun_out/${TAG}_ncu_k13.log 2>&1
echo "ncu k1/k3 rc=$?"
