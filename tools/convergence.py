"""The paper's accuracy study on the GPU right-hand side (Fig. 8).

Density wave on (0,2)^d: rho = 1 + 0.2 sin(pi sum x), v = (1,...,1), p = 1 translates with speed
(1,...,1); at T = 2 (one period) the exact solution equals the initial state.  Curved meshes with
the paper's sequential warp (reading R13).  h-refinement at fixed p and p-refinement at M = 4
for the entropy-conservative (EC) and entropy-stable (ES, LLF) schemes.

Error: the L2 norm of the density error computed with the degree-35 collapsed Gauss rule at
every element, from the modal solution evaluated in the kernels (es_eval_points: PKD basis, the element
map and its exact Jacobian at the rule's points).

Time integration: classical RK4 (R17; the paper uses DP8 with a step small enough that the time error
is negligible) at dt = CFL h / ((2p+1) max(|v| + c)), CFL = 0.1 by default; the time error of
RK4 at these steps is below the spatial error (checked with --cfl 0.05 in DESIGN.md section 6).

    python tools/convergence.py --dim 2 --p 4 5 --M 4 8 16 32 [--T 2] [--flux 0 1]
    python tools/convergence.py --dim 3 --p 1 2 3 4 5 6 --M 4 --flux 1          (p-refinement)
    python tools/convergence.py ... --nodes 1      (warp & blend mapping nodes)

Prints one JSON line per run and the observed orders log2(e_M / e_2M).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))

import quadrature as Q  # noqa: E402


def l2_density_error(ctx, torch, u, d, L, t, xi, wq):
    """sqrt(sum_e sum_q w_q J(xi_q) (rho_h - rho_exact(x_q, t))^2) with the rule (xi, wq)"""
    err2, jmin = 0.0, float("inf")
    chunk = max(1, int(2e8 // (ctx.nloc * (2 * d + 3))))  # points per pass (bounded device memory)
    for q0 in range(0, len(wq), chunk):
        xq, wc = xi[q0:q0 + chunk], wq[q0:q0 + chunk]
        npts = len(wc)
        x = torch.empty((ctx.nloc, npts, d), dtype=torch.float64, device="cuda")
        jac = torch.empty((ctx.nloc, npts), dtype=torch.float64, device="cuda")
        uq = ctx.eval_points(u, xq, x, jac)
        w = torch.from_numpy(np.ascontiguousarray(wc)).cuda()
        rho_ex = 1.0 + 0.2 * torch.sin(2.0 * math.pi / L * (x - t).sum(-1))
        err2 += float((w[None, :] * jac * (uq[..., 0] - rho_ex) ** 2).sum())
        jmin = min(jmin, float(jac.min()))
    return math.sqrt(err2), jmin


def run_case(es, I, torch, d, p, M, T, warp="paper", fm=1, cfl=0.1, rule_n=18, nodes=0):
    L = 2.0
    mesh = I.split_cartesian(d, M, L)
    w = {"paper": I.paper_warp(d, L), "bj": I.bj_warp(d, L, M), "none": None}[warp]
    ctx = es.Context(mesh, p, warp=w, interface_flux=fm, mapping_nodes=nodes)
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
    xi, wq = Q.collapsed_gauss_rule(d, rule_n)
    e0, _ = l2_density_error(ctx, torch, u, d, L, 0.0, xi, wq)
    t0 = time.perf_counter()
    ctx.set_state(u)
    ctx.step(dt, nsteps)
    ctx.get_state(u)
    ctx.synchronize()
    wall = time.perf_counter() - t0
    err, jmin = l2_density_error(ctx, torch, u, d, L, T, xi, wq)
    rate, scale, cons = ctx.entropy_production(u)
    ctx.close()
    return dict(dim=d, p=p, M=M, h=h, T=T, steps=nsteps, dt=dt, cfl=cfl, warp=warp, flux="ES" if fm else "EC",
                mapping_nodes=["lattice", "warp_and_blend"][nodes],
                l2_rho_error=err, l2_rho_error_t0=e0, min_jacobian=jmin, entropy_rate=rate, entropy_scale=scale,
                conservation=list(map(float, cons)), wall_s=wall, rule_degree=2 * rule_n - 1)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--dim", type=int, default=2)
    ap.add_argument("--p", type=int, nargs="+", default=[4, 5])
    ap.add_argument("--M", type=int, nargs="+", default=[4, 8, 16])
    ap.add_argument("--T", type=float, default=2.0)
    ap.add_argument("--cfl", type=float, default=0.1)
    ap.add_argument("--warp", default="paper", choices=["paper", "bj", "none"])
    ap.add_argument("--flux", type=int, nargs="+", default=[1, 0], help="1 = entropy stable (LLF), 0 = entropy conservative")
    ap.add_argument("--nodes", type=int, default=0, help="mapping nodes: 0 equispaced lattice (R10), 1 warp & blend (P:845, R32)")
    ap.add_argument("--out", default=None, help="JSONL file (appended)")
    args = ap.parse_args()
    import torch

    import es_inputs as I
    import paper_2312_07874_b200 as es
    out = open(args.out, "a") if args.out else None

    def emit(rec):
        line = json.dumps(rec)
        print(line, flush=True)
        if out:
            out.write(line + "\n")
            out.flush()
    for fm in args.flux:
        for p in args.p:
            errs = []
            for M in args.M:
                rec = run_case(es, I, torch, args.dim, p, M, args.T, args.warp, fm, args.cfl, nodes=args.nodes)
                errs.append(rec["l2_rho_error"])
                emit(rec)
            if len(args.M) > 1:
                orders = [math.log2(errs[k] / errs[k + 1]) * math.log(2) / math.log(args.M[k + 1] / args.M[k])
                          for k in range(len(errs) - 1)]
                emit({"dim": args.dim, "p": p, "flux": "ES" if fm else "EC", "M": args.M, "observed_orders": orders,
                      "expected": p + 1, "mapping_nodes": ["lattice", "warp_and_blend"][args.nodes]})


if __name__ == "__main__":
    main()
