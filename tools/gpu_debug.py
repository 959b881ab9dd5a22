"""Diagnostics on the GPU box: per-case relative errors vs the oracle (prints, never asserts)."""
import math
import sys
import time
import traceback

import numpy as np
import torch

sys.path.insert(0, ".")
import es_inputs as I
import oracle as O
import paper_2312_07874_b200 as es


def rel(a, b):
    return [float(np.abs(a[:, v] - b[:, v]).max() / max(np.abs(b[:, v]).max(), 1e-300)) for v in range(a.shape[1])]


def case(d, M, p, warp, ic, fm):
    L = 2.0 if d == 2 else 2 * math.pi
    mesh = I.split_cartesian(d, M, L)
    w = {"paper": I.paper_warp(d, L), "bj": I.bj_warp(d, L, M), "none": None}[warp]
    om = O.Mesh(mesh, p, warp=w)
    xq = om.node_coords()
    u0 = {"wave": lambda: I.density_wave(xq, L), "tgv": lambda: I.taylor_green(xq, 0.1),
          "tgv3": lambda: I.taylor_green(xq, 0.3), "vortex": lambda: I.isentropic_vortex(xq, L),
          "free": lambda: I.free_stream(xq, d)}[ic]()
    u = I.perturb_modal(om.project(u0), d, p, 1, 1e-2)
    ref, st = om.rhs(u, flux_mode=fm, variant=1)
    t = time.time()
    ctx = es.Context(mesh, p, warp=w, interface_flux=fm)
    ts = time.time() - t
    g = ctx.element_geometry(1)
    go = om.geometry(1)
    gerr = tuple(float(np.abs(g[k] - go[k]).max() / np.abs(go[k]).max()) for k in ("G", "Jn", "Jt"))
    ut = torch.from_numpy(u).cuda()
    du = torch.empty_like(ut)
    ctx.rhs(ut, du)
    ctx.synchronize()
    got = du.cpu().numpy()
    print(f"d={d} M={M} p={p} {warp} {ic} fm={fm}: setup {ts:.2f}s geo_err {gerr} rel {rel(got, ref)}", flush=True)
    if max(rel(got, ref)) > 1e-11:
        e = np.abs(got - ref).max(axis=(1, 2))
        print("   worst elements", np.argsort(-e)[:5], e[np.argsort(-e)[:5]], "ref scale", np.abs(ref).max())


for args in [(2, 3, 8, "bj", "vortex", 1), (2, 3, 10, "bj", "vortex", 1), (2, 3, 10, "paper", "wave", 1),
             (3, 3, 6, "paper", "tgv3", 1), (3, 3, 7, "paper", "tgv3", 1), (3, 3, 8, "bj", "tgv", 1),
             (3, 3, 8, "paper", "tgv", 1), (3, 4, 8, "bj", "tgv", 0)]:
    try:
        case(*args)
    except Exception:
        traceback.print_exc()
