#!/bin/bash
# K2 configuration sweep on C5: warps per CTA and volume jobs per flux batch.
# usage: K2CFGS="16,2 16,3 12,2" bash tools/gpu_k2sweep.sh   (pairs NWMAX,VB)
mkdir -p gpurun_out
for cfg in ${K2CFGS:-16,2 16,3 12,2 12,3 14,2}; do
  IFS=, read -r NW VB <<< "$cfg"
  export ES_NVCC_DEFS="-DES_K2_NWMAX=$NW -DES_K2_VB=$VB"
  touch paper_2312_07874_b200/csrc/rhs2.cuh
  python tools/build.py > gpurun_out/k2sw_build_${NW}_${VB}.log 2>&1 || { echo build fail $cfg; continue; }
  grep -A3 "rhs2_kernelILi3ELi9" build/kernels_3d.cu.o.log | grep -E "registers|spill" | head -2
  timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "rhs_parity and (3-3-8 or 3-3-5)" > gpurun_out/k2sw_pt_${NW}_${VB}.log 2>&1; echo "cfg $cfg pytest rc=$?"
  timeout 600 python bench.py --config C5 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/k2sw_${NW}_${VB}.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/k2sw_${NW}_${VB}.json')); k=d['roofline']['kernels']
print('cfg $cfg', 'ms/step %.2f'%d['ms_per_step'], 'K2 %.2f ms %.3f'%(k['K2']['ms_avg'], k['K2']['frac']))"
done
