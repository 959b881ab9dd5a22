#!/bin/bash
# K1 threads per CTA for tetrahedra at N = 9 (ES_K1_NT9). usage: NTS="320 352 416" bash tools/gpu_k1sweep.sh
mkdir -p gpurun_out
for NT in ${NTS:-320 352 416}; do
  export ES_NVCC_DEFS="-DES_K1_NT9=$NT"
  touch paper_2312_07874_b200/csrc/kernels.cuh
  python tools/build.py > gpurun_out/k1nt_build_$NT.log 2>&1 || { echo build fail $NT; continue; }
  grep -A3 "project_kernelILi3ELi9" build/kernels_3d.cu.o.log | grep -E "registers|spill" | head -2
  timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "rhs_parity and (3-3-8 or 3-4-8)" > gpurun_out/k1nt_pt_$NT.log 2>&1; echo "NT $NT pytest rc=$?"
  timeout 600 python bench.py --config C5 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/k1nt_$NT.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/k1nt_$NT.json')); k=d['roofline']['kernels']
print('NT $NT', 'ms/step %.2f'%d['ms_per_step'], 'K1 %.2f ms %.3f'%(k['K1']['ms_avg'], k['K1']['frac']))"
done
