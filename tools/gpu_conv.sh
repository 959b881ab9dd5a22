#!/bin/bash
# The paper's accuracy study on the GPU path: h- and p-refinement, EC and ES, T = 2.
mkdir -p gpurun_out
python tools/build.py > gpurun_out/conv_build.log 2>&1 || exit 1
timeout 600 python -m pytest tests/test_gpu_convergence.py -q -x > gpurun_out/conv_pytest.log 2>&1; tail -2 gpurun_out/conv_pytest.log
O=gpurun_out/r02_density_wave_convergence.jsonl
rm -f $O
timeout 900 python tools/convergence.py --dim 2 --p 2 3 4 5 --M 4 8 16 32 --flux 1 0 --out $O > /dev/null 2>gpurun_out/conv_2d.err
timeout 600 python tools/convergence.py --dim 2 --p 1 2 3 4 5 6 7 8 9 10 --M 4 --flux 1 0 --out $O > /dev/null 2>>gpurun_out/conv_2d.err
timeout 1800 python tools/convergence.py --dim 3 --p 4 5 --M 4 8 16 --flux 1 0 --out $O > /dev/null 2>gpurun_out/conv_3d.err
timeout 900 python tools/convergence.py --dim 3 --p 1 2 3 4 5 6 7 8 --M 4 --flux 1 0 --out $O > /dev/null 2>>gpurun_out/conv_3d.err
grep observed $O
