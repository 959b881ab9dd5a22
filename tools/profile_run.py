"""Small driver for ncu: C5-shaped element work (tet p=8, TGV, ES) on an M^3 x 6 mesh."""
import math
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import es_inputs as I
import paper_2312_07874_b200 as es

d = int(sys.argv[1]) if len(sys.argv) > 1 else 3
M = int(sys.argv[2]) if len(sys.argv) > 2 else 12
p = int(sys.argv[3]) if len(sys.argv) > 3 else 8
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 3
L = 2 * math.pi if d == 3 else 2.0
mesh = I.split_cartesian(d, M, L)
ctx = es.Context(mesh, p, warp=I.bj_warp(d, L, M), interface_flux=1)
u = torch.from_numpy(I.modal_state_from_centroids(mesh, p, "tgv" if d == 3 else "vortex", seed=1)).cuda()
du = torch.empty_like(u)
for _ in range(reps):
    ctx.rhs(u, du)
ctx.synchronize()
print("ok", float(du.abs().max()))
