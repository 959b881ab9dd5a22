"""Small driver for ncu: the bench workload's element work (projected analytic initial state) on a
smaller mesh.  usage: python tools/profile_run.py [dim M p reps [metric_storage]]"""
import math
import sys

import torch

sys.path.insert(0, ".")
import bench
import es_inputs as I
import paper_2312_07874_b200 as es

d = int(sys.argv[1]) if len(sys.argv) > 1 else 3
M = int(sys.argv[2]) if len(sys.argv) > 2 else 12
p = int(sys.argv[3]) if len(sys.argv) > 3 else 8
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 3
ms = int(sys.argv[5]) if len(sys.argv) > 5 else 0
L = 2 * math.pi if d == 3 else 2.0
mesh = I.split_cartesian(d, M, L)
ctx = es.Context(mesh, p, warp=I.bj_warp(d, L, M), interface_flux=1, metric_storage=ms)
u, xn, un = bench.initial_state(ctx, torch, "tgv" if d == 3 else "vortex", d, L)
du = torch.empty_like(u)
for _ in range(reps):
    ctx.rhs(u, du)
ctx.synchronize()
print("ok", float(du.abs().max()))
