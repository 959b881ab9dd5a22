#!/bin/bash
# The accuracy study on warp & blend mapping nodes (R32): density wave to T = 2, ES (and EC at p = 4).
mkdir -p gpurun_out
O=gpurun_out/wb_convergence.jsonl
rm -f $O
timeout 1500 python tools/convergence.py --dim 2 --p 2 3 4 5 --M 4 8 16 32 --flux 1 --nodes 1 --out $O > /dev/null 2>&1
timeout 600 python tools/convergence.py --dim 2 --p 4 --M 4 8 16 32 --flux 0 --nodes 1 --out $O > /dev/null 2>&1
timeout 1800 python tools/convergence.py --dim 3 --p 4 5 --M 4 8 16 --flux 1 --nodes 1 --out $O > /dev/null 2>&1
grep observed $O
