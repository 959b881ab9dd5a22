nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -O3 -I include -I paper_2312_07874_b200/csrc -o /tmp/dmma_psi1 tools/dmma_psi1.cu && /tmp/dmma_psi1 > gpurun_out/r02_dmma_psi1.jsonl; cat gpurun_out/r02_dmma_psi1.jsonl
python tools/build.py > /dev/null 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -q -k erk > gpurun_out/erk_pytest.log 2>&1; tail -2 gpurun_out/erk_pytest.log
for nt in 448 512; do
  export ES_NVCC_DEFS="-DES_K1_NT9=$nt"
  touch paper_2312_07874_b200/csrc/kernels.cuh
  python tools/build.py > gpurun_out/k1nt_build_$nt.log 2>&1 || { echo build fail; continue; }
  grep -A3 "project_kernelILi3ELi9" build/kernels_3d.cu.o.log | grep -E "registers|spill" | head -2
  timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "rhs_parity and 3-3-8" > gpurun_out/k1nt_pt_$nt.log 2>&1; echo "nt $nt pytest rc=$?"
  timeout 600 python bench.py --config C5 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/k1nt_$nt.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/k1nt_$nt.json')); k=d['roofline']['kernels']
print('nt $nt', 'ms/step %.2f'%d['ms_per_step'], 'K1 %.2f ms %.3f'%(k['K1']['ms_avg'], k['K1']['frac']))"
done
