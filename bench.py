#!/usr/bin/env python
"""Benchmark of the B200-native ES modal DSEM right-hand side (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C5] [--impl reference]

A *step* is one classical RK4 step of the whole hot path (4 right-hand sides: entropy projection,
line-wise flux differencing, facet correction, interface flux, lifting, weight-adjusted inverse,
fused stage update) over the configuration's mesh.  The default workload is BASELINE.json config
C5: 3D Euler, curved tetrahedra, p = 8, 32^3 x 6 = 196 608 elements, Taylor-Green vortex Ma 0.1,
entropy-stable interface flux.  Multi-GPU (torchrun): elements are partitioned into contiguous
slabs, face-trace halos go over NCCL; the timing is the max over ranks (CUDA events).

value = EC two-point flux evaluations per second, whole job (line-wise volume + facet-correction
pairs actually evaluated).  DOF.RHS/s and the Eq.-num_fluxes-equivalent rate
are reported alongside.  Inputs are synthetic (analytic initial data projected by the library).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # name: (dim, M, p, L, warp, initial state, interface flux, description)
    "C1": (2, 4, 2, 1.0, "none", "vortex", 1, "2D Euler p=2 affine triangles, 32 elements, isentropic vortex, ES"),
    "C2": (2, 32, 4, 2.0, "bj", "density_wave", 1, "2D Euler p=4 curved triangles, 2048 elements, density wave, ES"),
    "C3": (2, 64, 10, 2.0, "bj", "vortex", 1, "2D Euler p=10 curved triangles, 8192 elements, isentropic vortex, ES"),
    "C4": (3, 16, 4, 2 * math.pi, "bj", "tgv", 0, "3D Euler p=4 curved tetrahedra, 24576 elements, TGV Ma0.1, EC"),
    "C5": (3, 32, 8, 2 * math.pi, "bj", "tgv", 1,
           "3D Euler p=8 curved tetrahedra, 196608 elements, TGV Ma0.1, ES, RK4 step"),
}

# ---- algorithmic FP64 operation counts: +,-,*,/,sqrt,log,exp = 1 flop ----
FLUX_FLOPS = {2: 67, 3: 81}            # Ranocha EC flux, Taylor branch of both log means
VOL_NORMAL_FLOPS = {2: 12, 3: 24}      # n_ij from the line operators and averaged metrics
FAC_NORMAL_FLOPS = {2: 10, 3: 21}      # <J n> of the facet correction
ACC_FLOPS = {2: 8, 3: 10}              # -F to node i, +F to node j (or C^T 1)
IFACE_FLOPS = {2: 110, 3: 140}         # EC flux + Davis wave speed + LF jump + B J_f scaling (iface kernel)


def counts(dim, p):
    n = p + 1
    if dim == 2:
        vol, fac, eq56 = p * n * n, 3 * n * n, 3 * n * n * (p + 2) // 2
        iface = 3 * n
        Np, Nq = n * (n + 1) // 2, n * n
        sf = Np * n + n * n * n  # MACs per sum-factorised V (or V^T) apply, one variable
    else:
        vol, fac, eq56 = 3 * p * n ** 3 // 2, 3 * n ** 3 + n ** 4, 4 * n ** 4
        iface = 4 * n * n
        Np, Nq = n * (n + 1) * (n + 2) // 6, n ** 3
        sf = Np * n + (n * (n + 1) // 2) * n * n + n ** 4
    return dict(vol=vol, fac=fac, eq56=eq56, iface=iface, Np=Np, Nq=Nq, sf=sf)


def rhs_kernel_flops(dim, p, vol=None, fac=None):
    """algorithmic flops of the flux-differencing kernel (K2) per element and RHS: volume and
    facet-correction pairs, C^T 1 subtraction, lifting and the weight-adjusted inverse (the
    interface flux runs in its own kernel)"""
    c = counts(dim, p)
    nc = dim + 2
    f = (vol or c["vol"]) * (FLUX_FLOPS[dim] + VOL_NORMAL_FLOPS[dim] + ACC_FLOPS[dim])
    f += (fac or c["fac"]) * (FLUX_FLOPS[dim] + FAC_NORMAL_FLOPS[dim] + ACC_FLOPS[dim])
    if dim == 2:  # the 2D flux kernel also applies the weight-adjusted inverse (3D: K3, wadj_kernel_flops)
        f += 2 * 3 * nc * c["sf"]  # V^T, V, V^T of the weight-adjusted inverse
        f += nc * c["Nq"]  # W/J~ scaling
    f += nc * c["Nq"] * 2 * (dim + 1)  # lifting R^T s
    return f


def wadj_kernel_flops(dim, p):
    """algorithmic flops per element of the 3D weight-adjusted inverse kernel K3: three
    sum-factorised transforms V^T, V, V^T (2 flops per MAC, exact triangular loop bounds) and the
    W/J~ scaling"""
    c = counts(dim, p)
    nc = dim + 2
    return 2 * 3 * nc * c["sf"] + nc * c["Nq"]


def project_kernel_flops(dim, p):
    """algorithmic flops per element of the entropy-projection kernel K1: five
    sum-factorised transforms (V, V^T, V, V^T, V; 2 flops per multiply-add, exact loop bounds), the
    facet extrapolation, the entropy variables at the volume nodes (~35 flops each, logs and divisions
    counted as one) and the entropy-projected states at volume and facet nodes (~20 each)"""
    c = counts(dim, p)
    nc, n = dim + 2, p + 1
    nf = (dim + 1) * n ** (dim - 1)
    traces = 5 * n ** 3 if dim == 3 else 3 * n * n
    return 2 * 5 * nc * c["sf"] + 2 * nc * traces + 35 * c["Nq"] + 20 * (c["Nq"] + nf)


def iface_bytes_per_element(dim, p):
    """algorithmic HBM bytes per element of the interface kernel: own and neighbour traces (rho, v,
    p/2 at every facet node), J n at the facet nodes, B J_f f* written"""
    n = p + 1
    nf = (dim + 1) * n ** (dim - 1)
    nc = dim + 2
    return 8 * nf * (2 * nc + dim + nc)


def ncu_traffic_per_element(kernel="K2"):
    """DRAM bytes per element and launch of a kernel from the committed ncu --set full capture (profiles/)."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as fh:
            d = json.load(fh)
        key = {"K2": "rhs2_kernel", "K1": "project_kernel", "K3": "wadj3_kernel", "iface": "iface_kernel"}[kernel]
        return d[key]["dram_bytes_per_element"], d["source"]
    except Exception:
        return None, None


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return json.load(fh)
    except Exception:
        return {}


def fp64_peak_tflops(sm_mhz=None):
    """FP64 CUDA-core peak from the unit counts: 148 SMs x 64 DFMA/clk x 2 flop x clock
    (B200_PROFILING.md: 148 SMs, clocks.max.sm 1965 MHz)."""
    mhz = sm_mhz or measured_peaks().get("sm_max_mhz", 1965.0)
    return 148 * 64 * 2 * mhz * 1e6 / 1e12


# ------------------------------------------------------------------------------------------------
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region (200 ms)."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()
        sm, mx, reasons = [], 1965.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            try:
                sm.append(float(r[1]))
                mx = float(r[2])
                for k, nm in enumerate(names):
                    if r[5 + k].lower() in ("active", "yes", "1"):
                        reasons.add(nm)
            except Exception:
                continue
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


def _dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def initial_state(ctx, torch, kind, d, L):
    import es_inputs as I
    x = torch.empty((ctx.nloc, ctx.Nq, d), dtype=torch.float64, device="cuda")
    ctx.node_coords(x)
    ctx.synchronize()
    xn = x.cpu().numpy()
    un = {"tgv": lambda: I.taylor_green(xn, Ma=0.1), "density_wave": lambda: I.density_wave(xn, L),
          "vortex": lambda: I.isentropic_vortex(xn, L)}[kind]()
    um = torch.empty((ctx.nloc, d + 2, ctx.Np), dtype=torch.float64, device="cuda")
    ctx.project_nodal(torch.from_numpy(np.ascontiguousarray(un)).cuda(), um)
    ctx.synchronize()
    return um, xn, un


def cfl_dt(xn, un, d, L, M, p, cfl=0.1, gamma=1.4):
    """R16: dt = CFL h / ((2p+1) max(|v| + c)) from the initial nodal state, h = L/M."""
    rho = un[..., 0]
    v = un[..., 1:1 + d] / rho[..., None]
    pr = (gamma - 1) * (un[..., -1] - 0.5 * rho * np.sum(v * v, -1))
    smax = float(np.max(np.sqrt(np.sum(v * v, -1)) + np.sqrt(gamma * pr / rho)))
    return cfl * (L / M) / ((2 * p + 1) * smax)


def _oracle_sample(cfg, cores):
    """Set up the oracle (test infrastructure) on a bounded sample of configuration `cfg`: the
    elements of a compact block of mesh cells at the origin (2 x 2 x 2 cubes = 48 tetrahedra in 3D,
    5 x 5 squares = 50 triangles in 2D, or the whole mesh if smaller), so that the face neighbours
    whose geometry and entropy projection the oracle also needs stay few and setup stays at tens of
    seconds.  Returns (oracle mesh, modal state, sample, interface flux mode, number of elements)."""
    import es_inputs as I
    import oracle as O
    dim, M, p, L, warp, kind, fm, _ = CONFIGS[cfg]
    mesh = I.split_cartesian(dim, M, L)
    w = {"bj": I.bj_warp(dim, L, M), "none": None}.get(warp)
    u = I.modal_state_from_centroids(mesh, p, kind, seed=0, amp=1e-3)
    ne = len(mesh["elem_vertices"])
    b = min(M, 2 if dim == 3 else 5)
    per = 6 if dim == 3 else 2  # simplices per cell, consecutive in split_cartesian's order
    cells = [i + M * j + (M * M * k if dim == 3 else 0)
             for k in range(b if dim == 3 else 1) for j in range(b) for i in range(b)]
    sample = np.array(sorted(c * per + t for c in cells for t in range(per)), dtype=np.int64)
    om = O.Mesh(mesh, p, warp=w, active=sample)
    return om, u, sample, fm, ne


def _oracle_rhs(om, u, sample, fm, cores):
    """one oracle RHS on the sample; returns (seconds, flux evaluations)"""
    t0 = time.perf_counter()
    _, st = om.rhs(u, flux_mode=fm, variant=1, elems=sample, nthreads=cores)
    return time.perf_counter() - t0, st.volume_pairs + st.facet_pairs


def _sample_desc(cfg, nsample, ne, cores, reps):
    return (f"{cfg}: one oracle RHS (line-wise variant; entropy projection of the sample and its face "
            f"neighbours) on {nsample} of {ne} elements (a compact block of mesh cells), OpenMP {cores} "
            f"threads, mean of {reps}")


def _cpu_model():
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def cpu_baseline(cfg, budget_s=12.0):
    """The oracle as it stands (test infrastructure), timed on this host's cores on a bounded
    sample of the workload's elements, single-threaded and with all cores; returns
    flux evals/s of the oracle's line-wise RHS.  The sample is a compact block of cells: the oracle
    builds its geometry in extended precision at ~1 s per element and core at p = 8, so the 4096-element
    sample SURVEY 8(d) suggests would take about an hour of setup."""
    cores = os.cpu_count() or 1
    om, u, sample, fm, ne = _oracle_sample(cfg, cores)
    res = {}
    for nt in (1, cores):
        dt1, _ = _oracle_rhs(om, u, sample, fm, nt)
        reps = max(1, min(20, int(budget_s / 2 / max(dt1, 1e-3))))
        tot, evals = 0.0, 0
        for _ in range(reps):
            dt, evals = _oracle_rhs(om, u, sample, fm, nt)
            tot += dt
        res[nt] = (evals * reps / tot, tot / reps, reps)
    v_all, dt_all, reps = res[cores]
    return {"value": v_all, "unit": "flux_evals/s", "cores": cores, "kind": "oracle",
            "sample": _sample_desc(cfg, len(sample), ne, cores, reps), "seconds_per_rhs_sample": dt_all,
            "single_thread": {"value": res[1][0], "cores": 1, "seconds_per_rhs_sample": res[1][1]},
            "cpu_model": _cpu_model(),
            "flux_transform_split": "not instrumented (the oracle is timed as it stands, without internal timers)"}


def run_reference(args):
    """--impl reference: the CPU oracle as the reference arm, on this arm's config/metric/unit.
    The oracle is set up once on the bounded sample (untimed); each warm-up / timed step is one
    oracle RHS on that sample."""
    rank, world, _ = _dist_env()
    if rank != 0:
        return 0
    cfg = args.config
    cores = os.cpu_count() or 1
    om, u, sample, fm, ne = _oracle_sample(cfg, cores)
    for _ in range(args.warmup):
        _oracle_rhs(om, u, sample, fm, cores)
    tot, evals = 0.0, 0
    for _ in range(args.steps):
        dt, ev = _oracle_rhs(om, u, sample, fm, cores)
        tot += dt
        evals += ev
    value = evals / tot
    desc = _sample_desc(cfg, len(sample), ne, cores, args.steps)
    line = {"metric": "EC two-point flux evals/s", "value": value, "unit": "flux_evals/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": tot / args.steps * 1e3,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "impl": "reference",
            "config": {"workload": CONFIGS[cfg][7], "sample": desc},
            "cpu_baseline": {"value": value, "unit": "flux_evals/s", "cores": cores, "kind": "oracle",
                             "sample": desc},
            "e2e": {"value": value, "unit": "flux_evals/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def nccl_unique_id(dist, torch, rank, device):
    """rank 0 creates the 128-byte ncclUniqueId the library's communicator is built from
    (es_options.nccl_unique_id) and broadcasts it over the torch process group"""
    import ctypes
    lib = ctypes.CDLL("libnccl.so.2")
    uid = (ctypes.c_ubyte * 128)()  # opaque bytes, zeros included
    if rank == 0:
        assert lib.ncclGetUniqueId(ctypes.byref(uid)) == 0
    t = torch.tensor(list(bytes(uid)), dtype=torch.uint8, device=device)
    dist.broadcast(t, 0)
    return bytes(t.cpu().numpy().tobytes())


def run(args):
    import torch
    import torch.distributed as dist
    rank, world, local = _dist_env()
    if world != args.gpus:
        world = max(world, 1)
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import es_inputs as I
    import paper_2312_07874_b200 as es
    dim, M, p, L, warp, kind, fm, desc = CONFIGS[args.config]
    if args.p:
        p = args.p  # degree sweep on the same mesh (BASELINE C3: p = 2, 4, 6, 8, 10)
        desc = f"{desc} [degree override p={p}]"
    if args.interface_flux >= 0 and args.interface_flux != fm:
        fm = args.interface_flux
        desc = f"{desc} [interface flux {('EC', 'ES-LLF', 'ES-entropy-jump', 'ES-matrix')[fm]}]"
    mesh = I.split_cartesian(dim, M, L)
    w = {"bj": I.bj_warp(dim, L, M), "none": None}.get(warp)
    nccl_id = nccl_unique_id(dist, torch, rank, "cuda") if world > 1 else None
    stream = torch.cuda.Stream()
    t_setup = time.perf_counter()
    ctx = es.Context(mesh, p, warp=w, interface_flux=fm, rank=rank, world=world, nccl_id=nccl_id,
                     stream=stream.cuda_stream, device=local, volume_mode=args.volume_mode,
                     metric_storage=args.metric_storage)
    if args.metric_storage:
        desc = f"{desc} [modal metric storage: G = V g~ expanded in the flux kernel]"
    if args.volume_mode == 1:
        desc = f"{desc} [ablation: Eq. num_fluxes per-operator fluxes]"
    elif args.volume_mode == 2:
        desc = f"{desc} [ablation: brute force over all node pairs, dense operators]"
    t_setup = time.perf_counter() - t_setup
    um, xn, un = initial_state(ctx, torch, kind, dim, L)
    dt = cfl_dt(xn, un, dim, L, M, p)
    if world > 1:
        dtt = torch.tensor([dt], device="cuda", dtype=torch.float64)
        dist.all_reduce(dtt, op=dist.ReduceOp.MIN)
        dt = float(dtt.item())
    ctx.set_state(um)
    ctx.synchronize()
    c = counts(dim, p)
    fc = ctx.flux_counts()  # evaluations the kernels actually perform (volume_mode aware)
    assert (args.volume_mode == 2 or fc["facet"] == c["fac"]) and (args.volume_mode or fc["volume"] == c["vol"])
    c["vol"], c["fac"] = fc["volume"], fc["facet"]
    ne = len(mesh["elem_vertices"])

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    # warm-up
    with torch.cuda.stream(stream):
        for _ in range(args.warmup):
            ctx.step(dt, 1)
    ctx.synchronize()
    barrier()
    sampler = ClockSampler(local)
    sampler.start()
    ctx.reset_launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    # ---- timed region: K RK4 steps (CUDA-graph replays on one rank, es_set_graphs) ----
    e0.record(stream)
    for _ in range(args.steps):
        ctx.step(dt, 1)
    e1.record(stream)
    ctx.synchronize()
    barrier()
    clocks = sampler.stop()
    ms = e0.elapsed_time(e1)
    launches = ctx.launch_count()
    if world > 1:
        tt = torch.tensor([ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = float(tt[0].item())
    ms_step = ms / args.steps
    rhs_per_step = 4
    evals_step = rhs_per_step * ne * (c["vol"] + c["fac"])
    value = evals_step / (ms_step * 1e-3)
    dof = ne * c["Np"] * (dim + 2)
    # ---- per-kernel breakdown: the same K steps again, eager, CUDA events around every launch on the
    # context stream (the launching stream of all kernels) ----
    ctx.timing_enable(True)
    e4, e5 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e4.record(stream)
    for _ in range(args.steps):
        ctx.step(dt, 1)
    e5.record(stream)
    ctx.synchronize()
    eager_ms_step = e4.elapsed_time(e5) / args.steps
    kt = {}
    for cls, name in ((0, "K1"), (1, "K2"), (2, "iface"), (3, "K3")):
        tms, tn = ctx.timing_read(cls)
        kt[name] = (tms / max(tn, 1), tn / args.steps)  # ms per launch, launches per step
    ctx.timing_enable(False)
    # ---- end to end through the public C-ABI host-buffer call (es_step_host): every step copies the
    # state from pinned host memory to the device and the result back ----
    state = torch.empty_like(um)
    ctx.get_state(state)
    ctx.synchronize()
    host_in = state.cpu().pin_memory()
    host_out = torch.empty_like(host_in).pin_memory()
    barrier()
    esteps = max(1, min(args.steps, 3))
    t0 = time.perf_counter()
    for _ in range(esteps):
        ctx.step_host(host_in, host_out, dt, 1)
    e2e_ms = (time.perf_counter() - t0) * 1e3 / esteps
    barrier()
    if world > 1:
        tt = torch.tensor([e2e_ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e_ms = float(tt[0].item())
    e2e_value = evals_step / (e2e_ms * 1e-3)
    nbytes = host_in.numel() * 8
    # ---- roofline: each kernel against the bound that applies ----
    nloc = ne / world
    peak_fp64 = fp64_peak_tflops()
    hbm = measured_peaks().get("hbm_gbs", 6544.3)
    kernels = {}

    def add_alu(name, label, flops_el):
        ms_l, per_step = kt[name]
        if per_step == 0:
            return
        units = nloc * rhs_per_step / per_step  # elements per launch
        ach = flops_el * units / (ms_l * 1e-3) / 1e12
        kernels[name] = {"kernel": label, "bound": "alu", "ms_avg": ms_l, "launches_per_step": per_step,
                         "share_of_step": ms_l * per_step / eager_ms_step, "algorithmic_flops_per_element": flops_el,
                         "achieved": ach, "peak": peak_fp64, "unit": "TFLOP/s", "frac": ach / peak_fp64}
    add_alu("K2", "rhs2_kernel (line-wise flux differencing, facet correction, lifting)",
            rhs_kernel_flops(dim, p, c["vol"], c["fac"]))
    add_alu("K1", "project_kernel (entropy projection, traces)", project_kernel_flops(dim, p))
    if dim == 3:
        add_alu("K3", "wadj3_kernel (weight-adjusted inverse, RK update)", wadj_kernel_flops(dim, p))
    ms_f, per_f = kt["iface"]
    if per_f:
        b_el = iface_bytes_per_element(dim, p)
        ach = b_el * nloc * rhs_per_step / per_f / (ms_f * 1e-3) / 1e9
        kernels["iface"] = {"kernel": "iface_kernel (entropy-stable interface flux)", "bound": "hbm", "ms_avg": ms_f,
                            "launches_per_step": per_f, "share_of_step": ms_f * per_f / eager_ms_step,
                            "algorithmic_bytes_per_element": b_el, "achieved": ach, "peak": hbm, "unit": "GB/s",
                            "frac": ach / hbm}
    dom = max(kernels, key=lambda k: kernels[k]["share_of_step"])
    tpe, traffic_src = ncu_traffic_per_element(dom)
    k = kernels[dom]
    units = nloc * rhs_per_step / k["launches_per_step"]
    line = {
        "metric": "EC two-point flux evals/s", "value": value, "unit": "flux_evals/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"{args.config}: {desc}", "n_elements": ne, "p": p, "dim": dim,
                   "dof": dof, "dt": dt, "l2": "inputs larger than L2 (no flush needed)" if dof * 8 > 126e6 else
                   "inputs smaller than L2",
                   "parallelism": f"element partition over {world} GPU(s), NCCL face-trace halo",
                   "cuda_graphs": world == 1, "setup_s": t_setup},
        "dof_rhs_per_s": dof * rhs_per_step / (ms_step * 1e-3),
        "rhs_per_s": rhs_per_step / (ms_step * 1e-3),
        "eq56_equivalent_evals_per_s": rhs_per_step * ne * c["eq56"] / (ms_step * 1e-3),
        "roofline": {"bound": k["bound"], "achieved": k["achieved"], "peak": k["peak"], "unit": k["unit"],
                     "frac": k["frac"], "traffic": tpe * units if tpe else None, "kernel": k["kernel"],
                     "kernel_ms_avg": k["ms_avg"], "kernel_share_of_step": k["share_of_step"],
                     "traffic_source": traffic_src,
                     "peak_basis": ("148 SM x 64 DFMA/clk x 2 x sm_max_mhz (DESIGN.md 5.4)" if k["bound"] == "alu"
                                    else "MEASURED_PEAKS.json hbm_gbs"),
                     "eager_ms_per_step": eager_ms_step, "kernels": kernels},
        "e2e": {"value": e2e_value, "unit": "flux_evals/s", "h2d_bytes_per_step": nbytes, "d2h_bytes_per_step": nbytes,
                "api": "es_step_host (C ABI): pinned host state -> device, RK4 step, device -> pinned host"},
        "gpu_launches": int(launches),
        "clocks": clocks,
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            line["cpu_baseline"] = cpu_baseline(args.config)
            line["cpu_baseline"].pop("seconds_per_rhs_sample", None)
        except Exception as ex:  # pragma: no cover
            line["cpu_baseline"] = {"error": str(ex)}
    if rank == 0:
        print(json.dumps(line), flush=True)
    ctx.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C5", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--p", type=int, default=0, help="override the configuration's polynomial degree")
    ap.add_argument("--interface-flux", type=int, default=-1,
                    help="override the configuration's interface flux: 0 EC, 1 LLF, 2 entropy jump (R27), 3 matrix (R28)")
    ap.add_argument("--volume-mode", type=int, default=0,
                    help="1: ablation, one flux per operator S^(l) (the paper's Eq. num_fluxes iteration); "
                         "2: ablation, brute force over all node pairs (small configurations only)")
    ap.add_argument("--metric-storage", type=int, default=0,
                    help="1: modal (compressed) metric storage, PKD coefficients of G expanded in the flux kernel")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    return run(args)


if __name__ == "__main__":
    sys.exit(main())
