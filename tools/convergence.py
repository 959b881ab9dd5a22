"""Density-wave accuracy study on the GPU right-hand side (the paper's Fig. 8 experiment, P:885-922,
SURVEY 8(f) rank 1): rho = 1 + 0.2 sin(2 pi/L sum x), v = (1, ..., 1), p = 1 translates with speed
(1, ..., 1), so the exact solution at time T is the initial state shifted by T.  The L2
density error uses the physical quadrature weights W J~ of the volume nodes (es_node_weights) and
the nodal values u = V u~ (es_eval_nodal).  Time integration: classical RK4 (R17; the paper uses
DP8) at dt = CFL h / ((2p+1) max(|v| + c)) with a small CFL so that the spatial error dominates.

    python tools/convergence.py [--dim 2] [--p 2 3] [--M 4 8 16] [--T 0.2] [--warp paper|bj|none]

Prints one JSON line per (p, M) and the observed orders log2(e_M / e_2M).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def l2_density_error(ctx, torch, u, d, L, t):
    x = torch.empty((ctx.nloc, ctx.Nq, d), dtype=torch.float64, device="cuda")
    ctx.node_coords(x)
    un = torch.empty((ctx.nloc, ctx.Nq, d + 2), dtype=torch.float64, device="cuda")
    ctx.eval_nodal(u, un)
    wj = torch.empty((ctx.nloc, ctx.Nq), dtype=torch.float64, device="cuda")
    ctx.node_weights(wj)
    ctx.synchronize()
    rho_ex = 1.0 + 0.2 * torch.sin(2.0 * math.pi / L * (x - t).sum(-1))
    return math.sqrt(float((wj * (un[..., 0] - rho_ex) ** 2).sum()))


def run_case(es, I, torch, d, p, M, T, warp, fm=1, cfl=0.1):
    L = 2.0
    mesh = I.split_cartesian(d, M, L)
    w = {"paper": I.paper_warp(d, L), "bj": I.bj_warp(d, L, M), "none": None}[warp]
    ctx = es.Context(mesh, p, warp=w, interface_flux=fm)
    x = torch.empty((ctx.nloc, ctx.Nq, d), dtype=torch.float64, device="cuda")
    ctx.node_coords(x)
    ctx.synchronize()
    un = I.density_wave(x.cpu().numpy(), L)
    u = torch.empty((ctx.nloc, d + 2, ctx.Np), dtype=torch.float64, device="cuda")
    ctx.project_nodal(torch.from_numpy(np.ascontiguousarray(un)).cuda(), u)
    smax = math.sqrt(d) + math.sqrt(1.4 / 0.8)  # |v| + max c over the wave (rho >= 0.8, p = 1)
    h = L / M
    nsteps = int(math.ceil(T / (cfl * h / ((2 * p + 1) * smax))))
    dt = T / nsteps
    ctx.set_state(u)
    ctx.step(dt, nsteps)
    ctx.get_state(u)
    ctx.synchronize()
    err = l2_density_error(ctx, torch, u, d, L, T)
    ctx.close()
    return err, nsteps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--dim", type=int, default=2)
    ap.add_argument("--p", type=int, nargs="+", default=[2, 3])
    ap.add_argument("--M", type=int, nargs="+", default=[4, 8, 16])
    ap.add_argument("--T", type=float, default=0.2)
    ap.add_argument("--warp", default="paper", choices=["paper", "bj", "none"])
    ap.add_argument("--flux", type=int, default=1, help="1 = entropy stable (LLF), 0 = entropy conservative")
    args = ap.parse_args()
    import torch

    import es_inputs as I
    import paper_2312_07874_b200 as es
    for p in args.p:
        errs = []
        for M in args.M:
            e, n = run_case(es, I, torch, args.dim, p, M, args.T, args.warp, args.flux)
            errs.append(e)
            print(json.dumps({"dim": args.dim, "p": p, "M": M, "h": 2.0 / M, "steps": n, "T": args.T,
                              "warp": args.warp, "flux": "ES" if args.flux else "EC", "l2_rho_error": e}), flush=True)
        orders = [math.log2(errs[k] / errs[k + 1]) for k in range(len(errs) - 1)]
        print(json.dumps({"dim": args.dim, "p": p, "observed_orders": orders, "expected": p + 1}), flush=True)


if __name__ == "__main__":
    main()
