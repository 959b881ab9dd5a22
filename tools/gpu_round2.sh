#!/bin/bash
# Round-2 GPU pass: build, GPU tests, smoke, default bench (with the CPU baseline), the reference arm,
# all-configuration bench lines, ncu launch list of the bench command, ncu --set full of K1/K2/K3.
TAG=${1:-r02}
mkdir -p gpurun_out
python tools/build.py > gpurun_out/${TAG}_build.log 2>&1 || { echo build failed; exit 1; }
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${TAG}_gpu.txt 2>&1
lscpu > gpurun_out/${TAG}_lscpu.txt 2>&1; nproc >> gpurun_out/${TAG}_lscpu.txt
if [ "$2" != "skip-tests" ]; then
  timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/${TAG}_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest_gpu.log
  tail -3 gpurun_out/${TAG}_pytest_gpu.log
  timeout 300 python __graft_entry__.py smoke > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/${TAG}_smoke.log
  tail -1 gpurun_out/${TAG}_smoke.log
fi
timeout 900 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/${TAG}_reference.json 2> gpurun_out/${TAG}_reference.err; echo "reference rc=$?"
rm -f gpurun_out/${TAG}_configs.jsonl
for C in C1 C2 C3 C4; do
  timeout 600 python bench.py --config $C --steps 5 --warmup 3 --no-cpu-baseline >> gpurun_out/${TAG}_configs.jsonl 2>/dev/null
done
for P in 2 4 6 8; do
  timeout 600 python bench.py --config C3 --p $P --steps 5 --warmup 3 --no-cpu-baseline >> gpurun_out/${TAG}_configs.jsonl 2>/dev/null
done
timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_ncu_launch.log 2>&1
echo "launch list rc=$?"
timeout 300 python tools/profile_run.py 3 12 8 2 > gpurun_out/${TAG}_prof_plain.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"rhs2_kernel|project_kernel|wadj3" -s 3 -c 3 \
  -o gpurun_out/${TAG}_prof python tools/profile_run.py 3 12 8 2 > gpurun_out/${TAG}_ncu_full.log 2>&1
echo "ncu full rc=$?"
