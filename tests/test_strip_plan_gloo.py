"""Host logic of the strip partition on CPU
with world_size 2 and 3 over torch.distributed gloo: each rank plans its strip
through the C ABI (wrmg_plan_strip, no device), the ranks exchange their plans,
and the halo pattern is exercised with gloo point-to-point messages carrying
global column ids in place of the NCCL halo payload."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, gnx, gny, k, out):
    import torch
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2407_13997_b200 as w
        info, pv = w.wrmg_plan_strip(gnx, gny, 1.0 / gny, k, rank, world)
        plans = [None] * world
        dist.all_gather_object(plans, (info, pv.tolist()))
        # halo forward with gloo: every local column carries its global column id
        Lx = info["Lx"]
        v = np.full(Lx, -1.0)
        v[info["own0"]:info["own1"] + 1] = info["G0"] + np.arange(info["own0"], info["own1"] + 1)
        reqs, bufs = [], {}
        if info["nsl"]:
            reqs.append(dist.isend(torch.tensor(v[info["sl0"]:info["sl0"] + info["nsl"]]), rank - 1))
            bufs["L"] = torch.zeros(info["nlg"], dtype=torch.float64)
            reqs.append(dist.irecv(bufs["L"], rank - 1))
        if info["nsr"]:
            reqs.append(dist.isend(torch.tensor(v[info["sr0"]:info["sr0"] + info["nsr"]]), rank + 1))
            bufs["R"] = torch.zeros(info["nrg"], dtype=torch.float64)
            reqs.append(dist.irecv(bufs["R"], rank + 1))
        for r in reqs:
            r.wait()
        if "L" in bufs:
            v[info["lg0"]:info["lg0"] + info["nlg"]] = bufs["L"].numpy()
        if "R" in bufs:
            v[info["rg0"]:info["rg0"] + info["nrg"]] = bufs["R"].numpy()
        ghosts = [(c, v[c]) for c in list(range(info["lg0"], info["lg0"] + info["nlg"]))
                  + list(range(info["rg0"], info["rg0"] + info["nrg"]))]
        halo = [None] * world
        dist.all_gather_object(halo, (info["G0"], ghosts))
        if rank == 0:
            out.put((plans, halo))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,snx,gny,k", [(2, 6, 5, 2), (3, 4, 4, 3), (2, 4, 6, 1)])
def test_strip_plans_and_halo_over_gloo(world, snx, gny, k):
    from oracle import mesh, patches
    gnx = world * snx
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, gnx, gny, k, q)) for r in range(world)]
    for p in procs:
        p.start()
    plans, halo = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # owned columns partition the global lattice columns [0, k gnx]
    owned = []
    for info, _ in plans:
        owned += list(range(info["G0"] + info["own0"], info["G0"] + info["own1"] + 1))
    assert owned == list(range(k * gnx + 1))
    # ghosts received the owners' global column ids, and are exactly one cell wide
    for r, (G0, ghosts) in enumerate(halo):
        for c, val in ghosts:
            assert val == G0 + c
        assert len(ghosts) == k * ((r > 0) + (r < world - 1))
    # owned patches: disjoint, and together the global vertex-star patch set (R8)
    m = mesh.Mesh(gnx, gny, 1.0 / gny)
    _, verts = patches.vertex_star_patches(m, k, mesh.boundary_nodes(m, k))
    allv = np.concatenate([np.array(pv, dtype=np.int64) for _, pv in plans])
    assert len(allv) == len(set(allv.tolist()))
    assert sorted(allv.tolist()) == sorted(int(v) for v in verts)



def test_nccl_transport_loads_and_creates_unique_ids():
    """The NCCL transport of the strips (comm.cu) opens libnccl.so.2 at run time;
    rank 0's unique id is 128 bytes and differs between calls (no device needed)."""
    import paper_2407_13997_b200 as w
    a, b = w.nccl_unique_id(), w.nccl_unique_id()
    assert len(a) == 128 and len(b) == 128 and a != b and any(a)


def _ns_worker(rank, world, port, gnx, gny, k, out):
    import torch
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2407_13997_b200 as w
        iu, ip, pv, ps = w.wrmg_plan_ns_strip(gnx, gny, 1.0 / gny, k, rank, world)
        plans = [None] * world
        dist.all_gather_object(plans, (iu, ip, pv.tolist(), ps.tolist()))
        # halo forward of each lattice with gloo: every column carries its global id
        ghosts = []
        for info in (iu, ip):
            Lx = info["Lx"]
            v = np.full(Lx, -1.0)
            v[info["own0"]:info["own1"] + 1] = info["G0"] + np.arange(info["own0"], info["own1"] + 1)
            reqs, bufs = [], {}
            if info["nsl"]:
                reqs.append(dist.isend(torch.tensor(v[info["sl0"]:info["sl0"] + info["nsl"]]), rank - 1))
                bufs["L"] = torch.zeros(info["nlg"], dtype=torch.float64)
                reqs.append(dist.irecv(bufs["L"], rank - 1))
            if info["nsr"]:
                reqs.append(dist.isend(torch.tensor(v[info["sr0"]:info["sr0"] + info["nsr"]]), rank + 1))
                bufs["R"] = torch.zeros(info["nrg"], dtype=torch.float64)
                reqs.append(dist.irecv(bufs["R"], rank + 1))
            for r in reqs:
                r.wait()
            if "L" in bufs:
                v[info["lg0"]:info["lg0"] + info["nlg"]] = bufs["L"].numpy()
            if "R" in bufs:
                v[info["rg0"]:info["rg0"] + info["nrg"]] = bufs["R"].numpy()
            ghosts.append([(c, v[c]) for c in list(range(info["lg0"], info["lg0"] + info["nlg"]))
                           + list(range(info["rg0"], info["rg0"] + info["nrg"]))])
        halo = [None] * world
        dist.all_gather_object(halo, ghosts)
        if rank == 0:
            out.put((plans, halo))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,snx,gny,k", [(2, 4, 5, 1), (3, 3, 4, 2), (2, 2, 3, 2)])
def test_ns_strip_plans_and_halo_over_gloo(world, snx, gny, k):
    """Navier-Stokes strips: the owned columns of the velocity
    (degree k + 1) and pressure (degree k) lattices tile the global lattices, the
    gloo halo fills k + 1 / k ghost columns per side with the owners' columns, and
    the owned Vanka+star patches -- mapped back to global sids -- are exactly the
    oracle's patches (Fig. patches right), each on one rank."""
    from oracle import mesh, ns
    gnx = world * snx
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_ns_worker, args=(r, world, port, gnx, gny, k, q)) for r in range(world)]
    for p in procs:
        p.start()
    plans, halo = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for f, kk in ((0, k + 1), (1, k)):
        owned = []
        for pl in plans:
            info = pl[f]
            owned += list(range(info["G0"] + info["own0"], info["G0"] + info["own1"] + 1))
        assert owned == list(range(kk * gnx + 1))
        for r, gh in enumerate(halo):
            info = plans[r][f]
            for c, val in gh[f]:
                assert val == info["G0"] + c
            assert len(gh[f]) == kk * ((r > 0) + (r < world - 1))
    prob = ns.NSProblem(mesh.Mesh(gnx, gny, 1.0 / gny), k, 0, 1, 1.0, 1.0, bc="lid")
    pats, verts = ns.vanka_star_patches(prob)
    ref = {int(v): p.tolist() for v, p in zip(verts, pats)}
    got = {}
    for _, _, pv, ps in plans:
        for v, sids in zip(pv, ps):
            assert v not in got
            got[v] = [s for s in sids if s >= 0]
    assert got == ref
