set -x
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/fp64_pipes tools/fp64_pipes.cu && /tmp/fp64_pipes > gpurun_out/r02_fp64_pipes.json 2>&1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/fp64_micro tools/fp64_micro.cu && /tmp/fp64_micro > gpurun_out/r02_fp64_micro.json 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r02a_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02a_pytest_gpu.log
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/r02a_bench.json 2> gpurun_out/r02a_bench.err
lscpu > gpurun_out/r02_lscpu.txt; nproc >> gpurun_out/r02_lscpu.txt
