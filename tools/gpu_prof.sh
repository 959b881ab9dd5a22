#!/bin/bash
# ncu --set full of selected kernels on the profile_run workload (after a plain run exits 0).
# usage: bash tools/gpu_prof.sh TAG "kernel regex" [dim M p reps] [skip launches] [count]
TAG=$1; KRE=$2; shift 2
ARGS=${1:-"3 12 8 2"}
mkdir -p gpurun_out
python tools/build.py > gpurun_out/${TAG}_build.log 2>&1 || { echo build failed; exit 1; }
timeout 300 python tools/profile_run.py $ARGS > gpurun_out/${TAG}_prof_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$KRE" -s ${2:-2} -c ${3:-2} \
  -o gpurun_out/${TAG}_prof python tools/profile_run.py $ARGS > gpurun_out/${TAG}_ncu_full.log 2>&1
echo "ncu rc=$?"
