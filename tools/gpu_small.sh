#!/bin/bash
# Launch lists of the small configurations (kernel durations inside one RK4 step) + multirank tests.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_multirank.py -q -x > gpurun_out/sm_multirank.log 2>&1; echo "multirank rc=$?"; tail -1 gpurun_out/sm_multirank.log
for C in C1 C2; do
  timeout 300 python bench.py --config $C --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/sm_${C}.json 2>/dev/null && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/sm_${C}_launches.csv \
    python bench.py --config $C --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
  echo "$C rc=$?"
done
