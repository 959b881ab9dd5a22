#!/bin/bash
# modal metric storage on the GPU: parity tests, bench lines (C5, C4, C3) modal vs nodal, ncu of the
# modal flux kernel (DRAM bytes per element)
set -x
mkdir -p gpurun_out
python -m pytest tests/test_gpu_modal_metrics.py -q -x > gpurun_out/mm_pytest.log 2>&1; echo "pytest rc $?"
tail -3 gpurun_out/mm_pytest.log
for cfg in C5 C4 C3; do
  python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline --metric-storage 1 > gpurun_out/mm_bench_$cfg.json 2> gpurun_out/mm_bench_$cfg.err; echo "bench $cfg rc $?"
done
python bench.py --config C4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/nodal_bench_C4.json 2> gpurun_out/nodal_bench_C4.err
python bench.py --config C3 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/nodal_bench_C3.json 2> gpurun_out/nodal_bench_C3.err
python tools/profile_run.py 3 12 8 2 1 > gpurun_out/mm_prof_plain.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"rhs2_mm_kernel|rhs2_kernel" -s 1 -c 1 \
     -o gpurun_out/mm_prof -f python tools/profile_run.py 3 12 8 2 1 > gpurun_out/mm_ncu.log 2>&1; echo "ncu rc $?"
