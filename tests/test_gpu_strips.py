"""Strip partition of the heat hierarchy on
one GPU: nranks contexts driven by nranks host threads through the in-process
loopback transport (halo hand-over by host barrier + device copies; no kernel
waits on another rank).  Owned columns must match the single-rank global run."""
import threading

import numpy as np
import pytest

import wrmg_inputs as wi

pytestmark = pytest.mark.gpu


def _run_ranks(P, fn):
    out, err = [None] * P, []

    def body(r):
        try:
            out[r] = fn(r)
        except Exception as e:  # surfaced below
            err.append(e)

    th = [threading.Thread(target=body, args=(r,)) for r in range(P)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    if err:
        raise err[0]
    return out


def _owned(ctx, v):
    lay = ctx.layout
    Lx, NT = lay["lx"], lay["nt"]
    a = v.detach().cpu().numpy().reshape(lay["ly"], Lx, NT)
    return a[:, lay["own0"]:lay["own1"] + 1, :], lay["g0"] + lay["own0"]


@pytest.mark.parametrize("P,snx,ny,k,q,N,nc,bc", [(2, 8, 8, 2, 1, 6, 2, "dirichlet0"), (4, 4, 8, 1, 0, 5, 4, "dirichlet0"),
                                                (2, 8, 16, 3, 1, 3, 4, "dirichlet0"), (3, 8, 8, 2, 1, 40, 2, "dirichlet0"),
                                                # agglomerated coarse levels (strips narrower than 2 cells)
                                                (4, 4, 16, 2, 1, 6, 2, "dirichlet0"), (8, 4, 32, 3, 1, 4, 4, "dirichlet0"),
                                                (4, 2, 8, 1, 1, 33, 2, "dirichlet0"),
                                                # Neumann boundaries (the paper's heat runs)
                                                (2, 8, 8, 2, 1, 6, 2, "neumann"), (4, 4, 16, 3, 0, 5, 4, "neumann")])
def test_strips_match_global(P, snx, ny, k, q, N, nc, bc):
    import torch
    import paper_2407_13997_b200 as w
    gnx = P * snx
    h = 1.0 / ny
    dt = 1.0 / N
    # global single-rank reference on the same device
    g = w.Context(gnx, ny, h, degree=k, q=q, nslabs=N, dt=dt, ncoarse=nc, bc=bc)
    gl = g.layout
    f = wi.spacetime_field(gl["nnode"], N, q, 5)
    fd = torch.as_tensor(f, device="cuda:0")
    bg = g.empty()
    g.rhs(fd, bg)
    ug = g.zeros()
    g.smooth(ug, bg, 2, 1.0)
    rg = g.empty()
    g.residual(ug, bg, rg)
    zg = g.empty()
    g.vcycle(rg, zg)
    torch.cuda.synchronize()
    Lxg, NT = gl["lx"], gl["nt"]
    ref = {k2: v.cpu().numpy().reshape(gl["ly"], Lxg, NT) for k2, v in (("u", ug), ("r", rg), ("z", zg))}
    g.close()
    hub = w.LoopbackHub(P)

    def rank_fn(r):
        st = torch.cuda.Stream()
        with torch.cuda.stream(st):
            c = w.Context(gnx, ny, h, degree=k, q=q, nslabs=N, dt=dt, ncoarse=nc, rank=r, nranks=P, hub=hub,
                          stream=st.cuda_stream, bc=bc)
            lay = c.layout
            # f on the local lattice from the global generator (local column c <-> global g0 + c)
            Lx = lay["lx"]
            fl = f.reshape(gl["ly"], Lxg, NT)[:, lay["g0"]:lay["g0"] + Lx, :].copy()
            b = c.empty()
            c.rhs(torch.as_tensor(fl.reshape(-1), device="cuda:0"), b)
            u = c.zeros()
            c.smooth(u, b, 2, 1.0)
            rr = c.empty()
            c.residual(u, b, rr)
            z = c.empty()
            c.vcycle(rr, z)
            st.synchronize()
            res = {"u": _owned(c, u), "r": _owned(c, rr), "z": _owned(c, z)}
            c.close()
            return res

    outs = _run_ranks(P, rank_fn)
    hub.close()
    for key in ("u", "r", "z"):
        pieces = []
        for o in outs:
            a, c0 = o[key]
            pieces.append((c0, a))
        cols = sum(a.shape[1] for _, a in pieces)
        assert cols == Lxg
        full = np.concatenate([a for _, a in sorted(pieces, key=lambda x: x[0])], axis=1)
        e = np.linalg.norm(full - ref[key]) / np.linalg.norm(ref[key])
        assert e <= 1e-12, f"{key}: rel {e:.3e}"


@pytest.mark.parametrize("P,snx,ny,k,q,N,nc,bc", [(2, 8, 8, 2, 1, 6, 2, "dirichlet0"), (4, 4, 8, 1, 0, 5, 4, "dirichlet0"),
                                                (3, 8, 16, 3, 1, 4, 4, "dirichlet0"),
                                                # C2-shaped hierarchy (P3 x DG1, coarsest 4 x 4) split 4 and 8 ways:
                                                # the 4^2 and 8^2 levels run replicated
                                                (4, 8, 32, 3, 1, 16, 4, "dirichlet0"), (8, 4, 32, 3, 1, 16, 4, "dirichlet0"),
                                                (3, 8, 16, 2, 1, 4, 4, "neumann")])
def test_strips_fgmres_match_global(P, snx, ny, k, q, N, nc, bc):
    """FGMRES(30)-WRMG across strips (H13 with cross-rank dot products): the same
    iteration count as the single-rank solve and the owned columns of x equal to
    1e-9 (the sums run in a different order)."""
    import torch
    import paper_2407_13997_b200 as w
    gnx = P * snx
    h = 1.0 / ny
    dt = 1.0 / N
    g = w.Context(gnx, ny, h, degree=k, q=q, nslabs=N, dt=dt, ncoarse=nc, bc=bc)
    gl = g.layout
    f = wi.spacetime_field(gl["nnode"], N, q, 9)
    bg = g.empty()
    g.rhs(torch.as_tensor(f, device="cuda:0"), bg)
    xg = g.empty()
    its_g, rel_g, st_g = g.fgmres(bg, xg, restart=30, maxit=100, rtol=1e-10)
    torch.cuda.synchronize()
    Lxg, NT = gl["lx"], gl["nt"]
    ref = xg.cpu().numpy().reshape(gl["ly"], Lxg, NT)
    g.close()
    assert st_g == "WRMG_OK"
    hub = w.LoopbackHub(P)

    def rank_fn(r):
        st = torch.cuda.Stream()
        with torch.cuda.stream(st):
            c = w.Context(gnx, ny, h, degree=k, q=q, nslabs=N, dt=dt, ncoarse=nc, rank=r, nranks=P, hub=hub,
                          stream=st.cuda_stream, bc=bc)
            lay = c.layout
            Lx = lay["lx"]
            fl = f.reshape(gl["ly"], Lxg, NT)[:, lay["g0"]:lay["g0"] + Lx, :].copy()
            b = c.empty()
            c.rhs(torch.as_tensor(fl.reshape(-1), device="cuda:0"), b)
            x = c.empty()
            its, rel, status = c.fgmres(b, x, restart=30, maxit=100, rtol=1e-10)
            st.synchronize()
            res = (its, rel, status, _owned(c, x))
            c.close()
            return res

    outs = _run_ranks(P, rank_fn)
    hub.close()
    for its, rel, status, _ in outs:
        assert status == "WRMG_OK" and its == its_g, (its, its_g)
        assert rel == outs[0][1]  # identical on every rank
    full = np.concatenate([a for (a, c0) in sorted((o[3] for o in outs), key=lambda x: x[1])], axis=1)
    e = np.linalg.norm(full - ref) / np.linalg.norm(ref)
    assert e <= 1e-9, f"x: rel {e:.3e}"


@pytest.mark.parametrize("P,snx,ny,k,q,N,nc", [(2, 10, 20, 1, 1, 20, 10), (4, 10, 40, 2, 0, 20, 10),
                                             (4, 10, 40, 1, 3, 20, 10)])
def test_strips_paper_protocol_chebyshev(P, snx, ny, k, q, N, nc):
    """The paper's heat protocol (Neumann BCs, u0 = sin(pi x) + cos(2 pi y), T = 0.02, N = 20,
    Chebyshev-accelerated V(2,2) with lambda from 50 Arnoldi steps, FGMRES rtol/atol 1e-6;
    PAPER.md:366-379, 533-539) across strips: every rank's lambda equals the single-rank one
    (global dots), the FGMRES count is the single-rank count and x agrees on owned columns.
    The 40 x 40 meshes split 4 ways have 10 x 10 coarsest levels narrower than 2 cells per
    strip: they run replicated."""
    import torch
    import paper_2407_13997_b200 as w
    gnx = P * snx
    h = 1.0 / ny
    dt = 0.02 / N
    kw = dict(degree=k, q=q, nslabs=N, dt=dt, ncoarse=nc, bc="neumann", smoother="chebyshev", nu_pre=2, nu_post=2,
              weights="none")
    g = w.Context(gnx, ny, h, **kw)
    gl = g.layout
    u0 = wi.paper_heat_u0(gnx, ny, h, k)
    bg = g.zeros()  # wrmg_rhs_initial accumulates into b
    g.rhs_initial(torch.as_tensor(u0, device="cuda:0"), bg)
    xg = g.empty()
    its_g, rel_g, st_g = g.fgmres(bg, xg, restart=30, maxit=50, rtol=1e-6, atol=1e-6)
    lam_g = [g.cheb_lambda(l) for l in range(1, gl["nlevels"])]
    torch.cuda.synchronize()
    Lxg, NT = gl["lx"], gl["nt"]
    ref = xg.cpu().numpy().reshape(gl["ly"], Lxg, NT)
    g.close()
    assert st_g == "WRMG_OK"
    hub = w.LoopbackHub(P)
    Lx0 = k * gnx + 1

    def rank_fn(r):
        st = torch.cuda.Stream()
        with torch.cuda.stream(st):
            c = w.Context(gnx, ny, h, rank=r, nranks=P, hub=hub, stream=st.cuda_stream, **kw)
            lay = c.layout
            ul = u0.reshape(-1, Lx0)[:, lay["g0"]:lay["g0"] + lay["lx"]].copy().reshape(-1)
            b = c.zeros()
            c.rhs_initial(torch.as_tensor(ul, device="cuda:0"), b)
            x = c.empty()
            its, rel, status = c.fgmres(b, x, restart=30, maxit=50, rtol=1e-6, atol=1e-6)
            st.synchronize()
            res = (its, status, _owned(c, x))
            c.close()
            return res

    outs = _run_ranks(P, rank_fn)
    hub.close()
    for its, status, _ in outs:
        assert status == "WRMG_OK" and its == its_g, (its, its_g)
    full = np.concatenate([a for (a, c0) in sorted((o[2] for o in outs), key=lambda x: x[1])], axis=1)
    e = np.linalg.norm(full - ref) / np.linalg.norm(ref)
    assert e <= 1e-9, f"x: rel {e:.3e}"
    assert all(v > 0 for v in lam_g)
