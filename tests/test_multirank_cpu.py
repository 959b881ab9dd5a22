"""Multi-rank host logic on CPU (gloo, world size 2 and 3): the partition / face-halo plan of
es_plan driven through a real torch.distributed exchange.

Each rank fills its local face-trace slots with the global face id e*N_f + z, packs the slots of
es_plan's send list, exchanges them with gloo send/recv in the same grouped order the library
uses for NCCL (api.cu rhs_pass), and checks that every local face then finds, at its face_slot,
the global id of its neighbour face -- the one the single-rank plan names -- with the same
reflection flag.  No GPU is needed: es_plan is host-only.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import es_inputs as I


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, d, M, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2312_07874_b200 as es
        mesh = I.split_cartesian(d, M, 1.0)
        ev = mesh["elem_vertices"]
        nf = d + 1
        g = es.plan(d, ev, 0, 1)              # single-rank reference connectivity
        pl = es.plan(d, ev, rank, world)
        first, nloc = pl["first"], pl["nloc"]
        nslots = nloc * nf + pl["n_halo"]
        trace = torch.full((nslots,), -1.0, dtype=torch.float64)
        for k in range(nloc):
            for z in range(nf):
                trace[k * nf + z] = float((first + k) * nf + z)
        send = trace[torch.from_numpy(pl["send_slots"])] if len(pl["send_slots"]) else torch.zeros(0, dtype=torch.float64)
        soff = np.concatenate([[0], np.cumsum(pl["send_count"])])
        roff = np.concatenate([[0], np.cumsum(pl["recv_count"])])
        ops = []
        recv_bufs = {}
        for r in range(world):
            if r == rank:
                continue
            if pl["send_count"][r] > 0:
                ops.append(dist.P2POp(dist.isend, send[soff[r]:soff[r + 1]].contiguous(), r))
            if pl["recv_count"][r] > 0:
                buf = torch.empty(int(pl["recv_count"][r]), dtype=torch.float64)
                recv_bufs[r] = buf
                ops.append(dist.P2POp(dist.irecv, buf, r))
        if ops:
            for w in dist.batch_isend_irecv(ops):
                w.wait()
        for r, buf in recv_bufs.items():
            trace[nloc * nf + roff[r]: nloc * nf + roff[r + 1]] = buf
        # every local face finds its neighbour's trace
        bad = 0
        for k in range(nloc):
            e = first + k
            for z in range(nf):
                want = g["face_slot"][e, z]          # global slot o*Nf + zo in the 1-rank plan
                got = trace[pl["face_slot"][k, z]].item()
                bad += int(got != float(want))
                bad += int(pl["face_reflect"][k, z] != g["face_reflect"][e, z])
        # interior / boundary split: boundary elements are exactly those with a halo face
        halo = (pl["face_slot"] >= nloc * nf).any(axis=1)
        n_halo_faces = int((pl["face_slot"] >= nloc * nf).sum())
        tot = torch.tensor([bad, n_halo_faces, int(pl["send_count"].sum()), int(halo.sum())], dtype=torch.int64)
        gathered = [torch.zeros_like(tot) for _ in range(world)]
        dist.all_gather(gathered, tot)
        if rank == 0:
            allv = torch.stack(gathered)
            assert int(allv[:, 0].sum()) == 0, allv
            # faces received == faces sent, summed over ranks
            assert int(allv[:, 1].sum()) == int(allv[:, 2].sum()), allv
            if world > 1:
                assert int(allv[:, 3].min()) > 0
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("d,M,world", [(2, 4, 2), (3, 3, 2), (3, 4, 3)])
def test_halo_plan_exchange_gloo(d, M, world):
    pytest.importorskip("paper_2312_07874_b200")
    mp.spawn(_worker, args=(world, _free_port(), d, M, 0), nprocs=world, join=True)


def test_plan_partition_is_exhaustive():
    es = pytest.importorskip("paper_2312_07874_b200")
    mesh = I.split_cartesian(3, 4, 1.0)
    ev = mesh["elem_vertices"]
    ne = len(ev)
    for world in (1, 2, 4, 8):
        tot = 0
        sends = np.zeros((world, world), np.int64)
        recvs = np.zeros((world, world), np.int64)
        for r in range(world):
            pl = es.plan(3, ev, r, world)
            assert pl["first"] == tot
            tot += pl["nloc"]
            sends[r] = pl["send_count"]
            recvs[r] = pl["recv_count"]
            assert pl["send_count"][r] == 0 and pl["recv_count"][r] == 0
        assert tot == ne
        assert np.array_equal(sends, recvs.T)  # what r sends to s is what s expects from r


def _uid_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import bench
        uid = bench.nccl_unique_id(dist, torch, rank, "cpu")
        q.put((rank, uid))
    finally:
        dist.destroy_process_group()


def test_bench_nccl_unique_id_broadcast():
    # the id bytes (with zeros) reach every rank intact (bench.py multi-GPU setup path)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_uid_worker, args=(r, 2, port, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    got = dict(q.get(timeout=120) for _ in range(2))
    for pr in procs:
        pr.join(timeout=60)
    assert len(got[0]) == 128 and got[0] == got[1]
    assert got[0].count(0) > 0  # the id contains zero bytes that a C-string path would truncate
