#!/bin/bash
# Quick GPU iteration: selected GPU tests (pytest -k expression, or "all"), then short C5 / C4 bench lines.
# usage: bash tools/gpu_iter.sh TAG [pytest-k-expr|all|none] [bench configs...]
TAG=${1:-it}
K=${2:-all}
shift 2
mkdir -p gpurun_out
python tools/build.py > gpurun_out/${TAG}_build.log 2>&1 || { echo "build failed"; tail -20 gpurun_out/${TAG}_build.log; exit 1; }
if [ "$K" == "all" ]; then
  timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest_gpu.log
elif [ "$K" != "none" ]; then
  timeout 1500 python -m pytest tests -m gpu -x -q -k "$K" > gpurun_out/${TAG}_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest_gpu.log
fi
[ -f gpurun_out/${TAG}_pytest_gpu.log ] && tail -15 gpurun_out/${TAG}_pytest_gpu.log
for C in ${@:-C5}; do
  [ "$C" == "none" ] && continue
  timeout 600 python bench.py --config $C --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_bench_${C}.json 2> gpurun_out/${TAG}_bench_${C}.err
  echo "bench $C rc=$?"; python - <<PY
import json
try:
    d = json.load(open("gpurun_out/${TAG}_bench_${C}.json"))
    r = d["roofline"]; k = r["kernels"]
    print("$C", "ms/step %.2f" % d["ms_per_step"], "eager %.2f" % r["eager_ms_per_step"], "value %.3e" % d["value"],
          " ".join("%s %.2f ms %.3f" % (n, v["ms_avg"], v["frac"]) for n, v in k.items()), "e2e %.3e" % d["e2e"]["value"])
except Exception as ex:
    print("bench parse failed", ex); print(open("gpurun_out/${TAG}_bench_${C}.err").read()[-2000:])
PY
done
