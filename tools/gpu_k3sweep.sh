#!/bin/bash
# K3 configuration sweep: build each (threads, min blocks) variant, check 3D parity quickly, bench C5.
mkdir -p gpurun_out
for cfg in "256 1" "192 2" "384 1"; do
  set -- $cfg
  export ES_NVCC_DEFS="-DES_K3_THREADS=$1 -DES_K3_MINB=$2"
  touch paper_2312_07874_b200/csrc/xform3.cuh
  python tools/build.py > gpurun_out/sw_build_$1.log 2>&1 || { echo build fail; tail gpurun_out/sw_build_$1.log; continue; }
  timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "rhs_parity and (3-3-8 or 3-3-4 or 3-3-2) or entropy_production" > gpurun_out/sw_pytest_$1.log 2>&1; echo "cfg $cfg pytest rc=$?"; tail -2 gpurun_out/sw_pytest_$1.log
  timeout 600 python bench.py --config C5 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/sw_bench_$1.json 2>gpurun_out/sw_bench_$1.err
  python -c "
import json; d=json.load(open('gpurun_out/sw_bench_$1.json')); r=d['roofline']
print('cfg $cfg', 'ms/step %.2f'%d['ms_per_step'], 'K2 %.2f'%r['kernel_ms_avg'], 'K1 %.2f'%r['projection_kernel_ms_avg'], 'K3 %.2f ms %.2f TF'%(r['wadj_kernel_ms_avg'], r['wadj_tflops']))"
done
