"""Element partitioning on one GPU: R ranks' contexts in one
process, the face-trace halo moved by device-to-device copies through the two-stage RHS
(es_rhs_stage1 / es_halo_buffer / es_rhs_stage2) instead of NCCL.  The assembled d u~/dt must be
BITWISE equal to the single-rank result: per-element arithmetic does not depend on the partition.
Also checks the plan-driven halo against the oracle at the parity tolerance.
"""
import ctypes
import math

import numpy as np
import pytest

import es_inputs as I
import oracle as O

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def es():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2312_07874_b200 as es
    return es


def _cudart():
    lib = ctypes.CDLL("libcudart.so.12")
    lib.cudaMemcpy.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int]
    lib.cudaMemcpy.restype = ctypes.c_int
    lib.cudaDeviceSynchronize.restype = ctypes.c_int
    return lib


@pytest.mark.parametrize("d,M,p,world,fm", [(2, 4, 3, 2, 1), (2, 5, 4, 3, 0), (3, 3, 3, 3, 1), (3, 4, 4, 4, 1),
                                           (3, 3, 8, 2, 1)])
def test_multirank_loopback_bitwise(es, d, M, p, world, fm):
    L = 2.0 if d == 2 else 2.0 * math.pi
    mesh = I.split_cartesian(d, M, L)
    w = I.paper_warp(d, L)
    om = O.Mesh(mesh, p, warp=w)
    x = om.node_coords()
    u0 = I.density_wave(x, L) if d == 2 else I.taylor_green(x, Ma=0.3)
    u = I.perturb_modal(om.project(u0), d, p, seed=2, amp=1e-2)
    ev = mesh["elem_vertices"]
    ne = len(ev)
    # single rank
    ctx1 = es.Context(mesh, p, warp=w, interface_flux=fm)
    ut = torch.from_numpy(u).cuda()
    ref = torch.empty_like(ut)
    ctx1.rhs(ut, ref)
    ctx1.synchronize()
    ref = ref.cpu().numpy()
    # R ranks in this process
    rt = _cudart()
    ctxs, plans, ins, outs, sends = [], [], [], [], []
    for r in range(world):
        c = es.Context(mesh, p, warp=w, interface_flux=fm, rank=r, world=world, nccl_id=None)
        pl = es.plan(d, ev, r, world)
        assert c.first == pl["first"] and c.nloc == pl["nloc"]
        ctxs.append(c)
        plans.append(pl)
        ins.append(ut[pl["first"]:pl["first"] + pl["nloc"]].contiguous())
        outs.append(torch.empty_like(ins[-1]))
    for r, c in enumerate(ctxs):
        sends.append(c.rhs_stage1(ins[r]))
        c.synchronize()
    per_face = (d + 2) * ctxs[0].Nqf * 8  # bytes
    for r in range(world):
        soff = np.concatenate([[0], np.cumsum(plans[r]["send_count"])])
        for s in range(world):
            n = int(plans[r]["send_count"][s])
            if s == r or n == 0:
                continue
            roff = np.concatenate([[0], np.cumsum(plans[s]["recv_count"])])
            assert int(plans[s]["recv_count"][r]) == n
            dst = ctxs[s].halo_buffer() + int(roff[r]) * per_face
            src = sends[r] + int(soff[s]) * per_face
            assert rt.cudaMemcpy(dst, src, n * per_face, 3) == 0
    assert rt.cudaDeviceSynchronize() == 0
    for r, c in enumerate(ctxs):
        c.rhs_stage2(outs[r])
        c.synchronize()
    got = np.concatenate([o.cpu().numpy() for o in outs])
    assert got.shape == ref.shape and ne == got.shape[0]
    assert np.array_equal(got, ref)  # bitwise
    # and the oracle at the parity tolerance
    ora, _ = om.rhs(u, flux_mode=fm, variant=1)
    for v in range(d + 2):
        assert np.abs(got[:, v] - ora[:, v]).max() <= 1e-11 * np.abs(ora[:, v]).max()


def test_external_mode_requires_two_stage(es):
    mesh = I.split_cartesian(2, 4, 2.0)
    c = es.Context(mesh, 2, rank=0, world=2, nccl_id=None)
    u = torch.zeros(c.shape, dtype=torch.float64, device="cuda")
    with pytest.raises(es.ESError) as ex:
        c.rhs(u, torch.empty_like(u))
    assert ex.value.code == es.ES_ERR_CONFIG


@pytest.mark.parametrize("d,M,p,world,fm", [(2, 4, 3, 2, 1), (2, 5, 4, 3, 0), (3, 3, 3, 3, 1), (3, 4, 4, 4, 1),
                                           (3, 3, 8, 2, 1)])
def test_group_multirank_path_bitwise(es, d, M, p, world, fm):
    # es_group_*: the library's own world > 1 code path (pack, interior-element interface fluxes
    # overlapping the exchange on the communication stream, event ordering, boundary-element interface
    # fluxes, flux kernel, K3, RK4 stages, the reductions) with only the NCCL calls replaced by
    # device-to-device copies; bitwise equal to one rank
    L = 2.0 if d == 2 else 2.0 * math.pi
    mesh = I.split_cartesian(d, M, L)
    w = I.paper_warp(d, L)
    om = O.Mesh(mesh, p, warp=w)
    x = om.node_coords()
    u0 = I.density_wave(x, L) if d == 2 else I.taylor_green(x, Ma=0.3)
    u = I.perturb_modal(om.project(u0), d, p, seed=2, amp=1e-2)
    ut = torch.from_numpy(u).cuda()
    ctx1 = es.Context(mesh, p, warp=w, interface_flux=fm)
    ref = torch.empty_like(ut)
    ctx1.rhs(ut, ref)
    dt = 1e-3
    ctx1.set_state(ut)
    ctx1.step(dt, 3)
    ref_step = torch.empty_like(ut)
    ctx1.get_state(ref_step)
    rate1, sc1, cons1 = ctx1.entropy_production(ut)
    ctx1.synchronize()
    ctxs = [es.Context(mesh, p, warp=w, interface_flux=fm, rank=r, world=world, nccl_id=None) for r in range(world)]
    assert any(len(es.plan(d, mesh["elem_vertices"], r, world)["send_slots"]) for r in range(world))
    ins = [ut[c.first:c.first + c.nloc].contiguous() for c in ctxs]
    outs = [torch.empty_like(t) for t in ins]
    es.group_rhs(ctxs, ins, outs)
    for c in ctxs:
        c.synchronize()
    got = torch.cat(outs).cpu().numpy()
    assert np.array_equal(got, ref.cpu().numpy())  # bitwise
    # three RK4 steps on the library states, twice (the send buffers are reused across stages)
    for c, t in zip(ctxs, ins):
        c.set_state(t)
    es.group_step(ctxs, dt, 3)
    st = []
    for c, t in zip(ctxs, ins):
        o = torch.empty_like(t)
        c.get_state(o)
        c.synchronize()
        st.append(o)
    assert np.array_equal(torch.cat(st).cpu().numpy(), ref_step.cpu().numpy())
    # entropy production and conservation summed over ranks (the allreduce of es_entropy_production)
    rate, sc, cons = es.group_entropy_production(ctxs, ins)
    assert abs(rate - rate1) <= 1e-13 * sc1 and abs(sc - sc1) <= 1e-13 * sc1
    assert np.abs(cons - cons1).max() <= 1e-13 * max(np.abs(cons1).max(), sc1)
