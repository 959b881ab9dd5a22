#!/bin/bash
# Robustness runs of the paper swept over p = 4..8: KHI (2D, M = 16, T = 15) and the TGV at
# Ma = 0.7 (3D, M = 4, T = 14), EC and ES-LLF.
mkdir -p gpurun_out
python tools/build.py > gpurun_out/rob_build.log 2>&1 || exit 1
O=gpurun_out/r02_robustness_sweep.jsonl
rm -f $O
for p in 4 5 6 7 8; do
  timeout 900 python tools/robustness.py --case khi --p $p --M 16 --flux 0 1 --samples 15 >> $O 2>>gpurun_out/rob.err
  timeout 900 python tools/robustness.py --case tgv --Ma 0.7 --p $p --M 4 --flux 0 1 --samples 15 >> $O 2>>gpurun_out/rob.err
done
python -c "
import json
for l in open('$O'):
    d = json.loads(l); print(d['case'], d['p'], d['flux'], d['status'][:60], 't_end %.2f' % d['t_end'], 'dS %.3e' % d['history'][-1]['dS'])
"
