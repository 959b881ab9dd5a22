#!/bin/bash
# K3 configuration sweep (threads per CTA, resident CTAs per SM) on C5
mkdir -p gpurun_out
for cfg in "192 2" "96 4" "288 1" "384 1"; do
  set -- $cfg
  export ES_NVCC_DEFS="-DES_K3_THREADS=$1 -DES_K3_MINB=$2"
  touch paper_2312_07874_b200/csrc/xform3.cuh
  python tools/build.py > gpurun_out/k3sw_build_$1.log 2>&1 || { echo build fail; continue; }
  grep -A3 "wadj3_kernelILi9" build/xform3.cu.o.log | grep -E "registers|spill" | head -2
  timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "rhs_parity and (3-3-8 or 3-3-4-bj) or entropy_production and 3-" > gpurun_out/k3sw_pt_$1.log 2>&1; echo "cfg $cfg pytest rc=$?"
  timeout 600 python bench.py --config C5 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/k3sw_$1.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/k3sw_$1.json')); k=d['roofline']['kernels']
print('cfg $cfg', 'ms/step %.2f'%d['ms_per_step'], 'K3 %.2f ms %.3f'%(k['K3']['ms_avg'], k['K3']['frac']))"
done
