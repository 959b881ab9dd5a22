"""Entropy and conservation histories on the GPU path (the paper's robustness / entropy experiments,
P:924-926 and Fig. 9): the Taylor-Green vortex (R15) on
curved tetrahedra, integrated with es_step (classical RK4, R17) for EC and ES interface fluxes.
Records the total entropy  S(t) = sum W J~ s(u),  s = -rho (ln p - gamma ln rho)/(gamma - 1)
(P:820), its rate from es_entropy_production (sum w^T M~ du/dt), and the drift of the
conserved totals sum W J~ u.  EC: dS/dt = 0 to roundoff; ES: dS/dt <= 0.

    python tools/entropy_history.py [--M 4] [--p 3] [--Ma 0.1] [--steps 200] [--every 20] [--cfl 0.1]
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
GAMMA = 1.4


def totals(ctx, torch, u, d):
    un = torch.empty((ctx.nloc, ctx.Nq, d + 2), dtype=torch.float64, device="cuda")
    ctx.eval_nodal(u, un)
    wj = torch.empty((ctx.nloc, ctx.Nq), dtype=torch.float64, device="cuda")
    ctx.node_weights(wj)
    ctx.synchronize()
    rho = un[..., 0]
    ke = 0.5 * (un[..., 1:1 + d] ** 2).sum(-1) / rho
    p = (GAMMA - 1.0) * (un[..., -1] - ke)
    s = -rho * (torch.log(p) - GAMMA * torch.log(rho)) / (GAMMA - 1.0)
    S = float((wj * s).sum())
    cons = [float((wj * un[..., v]).sum()) for v in range(d + 2)]
    return S, cons


def run(es, I, torch, M, p, Ma, steps, every, fm, cfl=0.1, warp="bj"):
    d, L = 3, 2.0 * math.pi
    mesh = I.split_cartesian(d, M, L)
    w = I.bj_warp(d, L, M) if warp == "bj" else I.paper_warp(d, L)
    ctx = es.Context(mesh, p, warp=w, interface_flux=fm)
    x = torch.empty((ctx.nloc, ctx.Nq, d), dtype=torch.float64, device="cuda")
    ctx.node_coords(x)
    ctx.synchronize()
    un = I.taylor_green(x.cpu().numpy(), Ma=Ma)
    u = torch.empty((ctx.nloc, d + 2, ctx.Np), dtype=torch.float64, device="cuda")
    ctx.project_nodal(torch.from_numpy(np.ascontiguousarray(un)).cuda(), u)
    rho = un[..., 0]
    v = un[..., 1:4] / rho[..., None]
    pr = (GAMMA - 1) * (un[..., 4] - 0.5 * rho * (v * v).sum(-1))
    smax = float(np.max(np.sqrt((v * v).sum(-1)) + np.sqrt(GAMMA * pr / rho)))
    dt = cfl * (L / M) / ((2 * p + 1) * smax)
    ctx.set_state(u)
    out = []
    for k in range(0, steps + 1, every):
        if k:
            ctx.step(dt, every)
        ctx.get_state(u)
        ctx.synchronize()
        S, cons = totals(ctx, torch, u, d)
        rate, scale, _ = ctx.entropy_production(u)
        out.append({"t": k * dt, "step": k, "S": S, "dSdt": rate, "dSdt_scale": scale, "totals": cons})
    ctx.close()
    return out, dt


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--M", type=int, default=4)
    ap.add_argument("--p", type=int, default=3)
    ap.add_argument("--Ma", type=float, default=0.1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--every", type=int, default=20)
    ap.add_argument("--cfl", type=float, default=0.1)
    args = ap.parse_args()
    import torch

    import es_inputs as I
    import paper_2312_07874_b200 as es
    for fm, name in ((0, "EC"), (1, "ES")):
        hist, dt = run(es, I, torch, args.M, args.p, args.Ma, args.steps, args.every, fm, args.cfl)
        for h in hist:
            h.update({"flux": name, "M": args.M, "p": args.p, "Ma": args.Ma, "dt": dt})
            print(json.dumps(h), flush=True)


if __name__ == "__main__":
    main()
