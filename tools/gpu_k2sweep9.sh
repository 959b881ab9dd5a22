#!/bin/bash
# K2 warps per CTA for tetrahedra at N = 9 (ES_K2_NW9). usage: NWS="9 10 11 12 13" bash tools/gpu_k2sweep9.sh
mkdir -p gpurun_out
for NW in ${NWS:-9 10 11 13}; do
  export ES_NVCC_DEFS="-DES_K2_NW9=$NW"
  touch paper_2312_07874_b200/csrc/rhs2.cuh
  python tools/build.py > gpurun_out/k2n9_build_$NW.log 2>&1 || { echo build fail $NW; continue; }
  grep -A3 "rhs2_kernelILi3ELi9" build/kernels_3d.cu.o.log | grep -E "registers|spill" | head -2
  timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "rhs_parity and (3-3-8 or 3-4-8)" > gpurun_out/k2n9_pt_$NW.log 2>&1; echo "NW $NW pytest rc=$?"
  timeout 600 python bench.py --config C5 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/k2n9_$NW.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/k2n9_$NW.json')); k=d['roofline']['kernels']
print('NW $NW', 'ms/step %.2f'%d['ms_per_step'], 'K2 %.2f ms %.3f'%(k['K2']['ms_avg'], k['K2']['frac']))"
done
