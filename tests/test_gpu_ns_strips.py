"""Strip partition of the Navier-Stokes hierarchy (DESIGN.md section
7c) on one GPU: nranks contexts driven by nranks host threads through the
in-process loopback transport.  Each field (u_x, u_y on the velocity lattice, p on
the pressure lattice) is split by lattice columns; the owned columns of every
result must equal the single-rank global run on the same device.

The linearisation state is handed to each rank with only its OWNED columns
correct (every other local column is filled with junk): the library must rewrite
the rest from the owners (state refresh) before assembling the Vanka blocks."""
import numpy as np
import pytest

import wrmg_inputs as wi
from test_gpu_strips import _run_ranks

pytestmark = pytest.mark.gpu


def _fields(v, lay):
    """(u_x, u_y, p) views (Ly, Lx, NT) of an NS level vector."""
    NT, lx, ly, lu = lay["nt"], lay["lx"], lay["ly"], lay["lu"]
    a = np.asarray(v).reshape(-1, NT)
    return (a[:lu].reshape(ly, lx, NT), a[lu:2 * lu].reshape(ly, lx, NT),
            a[2 * lu:].reshape(lay["lpy"], lay["lpx"], NT))


def _window(vg, gl, lay, junk_seed=None):
    """The local vector of a rank cut from a global vector; junk_seed: every column
    the rank does not own is replaced by junk."""
    gu, gv, gp = _fields(vg, gl)
    out = []
    for f, (g, c0, o0, o1) in enumerate(((gu, lay["g0"], lay["own0"], lay["own1"]),
                                          (gv, lay["g0"], lay["own0"], lay["own1"]),
                                          (gp, lay["g0p"], lay["own0p"], lay["own1p"]))):
        lx = lay["lpx"] if f == 2 else lay["lx"]
        w = g[:, c0:c0 + lx, :].copy()
        if junk_seed is not None:
            rng = np.random.default_rng(junk_seed + f)
            mask = np.ones(lx, bool)
            mask[o0:o1 + 1] = False
            w[:, mask, :] = rng.uniform(-50, 50, size=w[:, mask, :].shape)
        out.append(w.reshape(-1))
    return np.concatenate(out)


def _owned(v, lay):
    fu, fv, fp = _fields(v, lay)
    o0, o1, q0, q1 = lay["own0"], lay["own1"], lay["own0p"], lay["own1p"]
    return ((lay["g0"] + o0, fu[:, o0:o1 + 1]), (lay["g0"] + o0, fv[:, o0:o1 + 1]),
            (lay["g0p"] + q0, fp[:, q0:q1 + 1]))


def _assemble(outs, key, gl):
    """Global field arrays from the ranks' owned columns (must tile the lattices)."""
    res = []
    for f in range(3):
        pieces = sorted((o[key][f] for o in outs), key=lambda x: x[0])
        full = np.concatenate([a for _, a in pieces], axis=1)
        res.append(full)
    assert res[0].shape[1] == gl["lx"] and res[2].shape[1] == gl["lpx"]
    return res


def _rel(a, b):
    return max(np.linalg.norm(x - y) / max(np.linalg.norm(y), 1e-300) for x, y in zip(a, b))


CASES = [  # P, snx, ny, k, q, N, ncoarse
    (2, 8, 16, 1, 1, 3, 2),
    (2, 8, 16, 2, 1, 3, 2),
    (3, 8, 24, 1, 0, 4, 3),
    (4, 4, 16, 2, 1, 2, 2),
]


@pytest.mark.parametrize("P,snx,ny,k,q,N,nc", CASES)
def test_ns_strips_match_global(P, snx, ny, k, q, N, nc):
    """Linearised at the C3 wind (R18): residual, nonlinear residual, two sweeps and
    one V(1,1) on the owned columns equal the single-rank run (1e-12)."""
    import torch
    import paper_2407_13997_b200 as w
    gnx = P * snx
    h = 1.0 / ny
    dt = 1.0 / N
    kw = dict(degree=k, q=q, nslabs=N, dt=dt, ncoarse=nc, problem="ns", reynolds=50.0, bc="lid", omega_mg=0.8)
    g = w.Context(gnx, ny, h, **kw)
    gl = g.layout
    W = wi.wind_state(gnx, ny, h, k, N, q, dt)
    f = wi.spacetime_field(gl["nnode"], N, q, 5)
    u0 = wi.spacetime_field(gl["nnode"], N, q, 6) * 0.1
    dev = lambda a: torch.as_tensor(a, device="cuda:0")
    g.linearize(dev(W))
    bg = g.empty()
    g.rhs(dev(f), bg)
    rg = g.empty()
    g.residual(dev(u0), bg, rg)
    nrg = g.empty()
    g.residual(dev(u0), bg, nrg, nonlinear=True)
    ug = dev(u0.copy())
    g.smooth(ug, bg, 2, 0.8)
    zg = g.empty()
    g.vcycle(rg, zg)
    torch.cuda.synchronize()
    ref = {key: _fields(v.cpu().numpy(), gl) for key, v in (("r", rg), ("nr", nrg), ("u", ug), ("z", zg))}
    g.close()
    hub = w.LoopbackHub(P)

    def rank_fn(r):
        st = torch.cuda.Stream()
        with torch.cuda.stream(st):
            c = w.Context(gnx, ny, h, rank=r, nranks=P, hub=hub, stream=st.cuda_stream, **kw)
            lay = c.layout
            assert lay["lu"] == lay["lx"] * lay["ly"]
            c.linearize(dev(_window(W, gl, lay, junk_seed=100 + r)))
            b = c.empty()
            c.rhs(dev(_window(f, gl, lay)), b)
            ul = _window(u0, gl, lay)
            rr = c.empty()
            c.residual(dev(ul), b, rr)
            nr = c.empty()
            c.residual(dev(ul), b, nr, nonlinear=True)
            u = dev(ul.copy())
            c.smooth(u, b, 2, 0.8)
            z = c.empty()
            c.vcycle(rr, z)
            st.synchronize()
            res = {key: _owned(v.cpu().numpy(), lay) for key, v in (("r", rr), ("nr", nr), ("u", u), ("z", z))}
            c.close()
            return res

    outs = _run_ranks(P, rank_fn)
    hub.close()
    for key in ("r", "nr", "u", "z"):
        e = _rel(_assemble(outs, key, gl), ref[key])
        assert e <= 1e-12, f"{key}: rel {e:.3e}"


@pytest.mark.parametrize("P,snx,ny,k,q,N,nc", [(2, 8, 16, 2, 1, 3, 2), (4, 4, 16, 1, 1, 4, 2)])
def test_ns_strips_fgmres(P, snx, ny, k, q, N, nc):
    """FGMRES(30)-WRMG on the Oseen system at the C3 wind: the single-rank iteration
    count on every rank and the owned columns of x equal to 1e-9."""
    import torch
    import paper_2407_13997_b200 as w
    gnx = P * snx
    h = 1.0 / ny
    dt = 0.05 / N
    kw = dict(degree=k, q=q, nslabs=N, dt=dt, ncoarse=nc, problem="ns", reynolds=20.0, bc="lid", omega_mg=0.8)
    dev = lambda a: torch.as_tensor(a, device="cuda:0")
    g = w.Context(gnx, ny, h, **kw)
    gl = g.layout
    W = wi.wind_state(gnx, ny, h, k, N, q, dt)
    f = wi.spacetime_field(gl["nnode"], N, q, 9)
    g.linearize(dev(W))
    bg = g.empty()
    g.rhs(dev(f), bg)
    xg = g.empty()
    its_g, rel_g, st_g = g.fgmres(bg, xg, restart=30, maxit=100, rtol=1e-8)
    torch.cuda.synchronize()
    ref = _fields(xg.cpu().numpy(), gl)
    g.close()
    assert st_g == "WRMG_OK"
    hub = w.LoopbackHub(P)

    def rank_fn(r):
        st = torch.cuda.Stream()
        with torch.cuda.stream(st):
            c = w.Context(gnx, ny, h, rank=r, nranks=P, hub=hub, stream=st.cuda_stream, **kw)
            lay = c.layout
            c.linearize(dev(_window(W, gl, lay, junk_seed=7 * r)))
            b = c.empty()
            c.rhs(dev(_window(f, gl, lay)), b)
            x = c.empty()
            its, rel, status = c.fgmres(b, x, restart=30, maxit=100, rtol=1e-8)
            st.synchronize()
            res = {"its": its, "rel": rel, "st": status, "x": _owned(x.cpu().numpy(), lay)}
            c.close()
            return res

    outs = _run_ranks(P, rank_fn)
    hub.close()
    for o in outs:
        assert o["st"] == "WRMG_OK" and o["its"] == its_g, (o["its"], its_g)
        assert o["rel"] == outs[0]["rel"]
    e = _rel(_assemble(outs, "x", gl), ref)
    assert e <= 1e-9, f"x: rel {e:.3e}"


@pytest.mark.parametrize("P,k,cheb", [(2, 1, False), (2, 2, False), (4, 1, True)])
def test_ns_strips_newton_cavity(P, k, cheb):
    """Newton-FGMRES-WRMG (R22) on the lid-driven cavity across
    strips (C4's protocol at a small size; cheb: Chebyshev V(2,2), lambda per level
    from global dot products): identical Newton and linear counts, U within 1e-8."""
    import torch
    import paper_2407_13997_b200 as w
    n, q, N, dt, R = 16, 1, 3, 0.05, 10.0
    kw = dict(degree=k, q=q, nslabs=N, dt=dt, ncoarse=2, problem="ns", reynolds=R, bc="lid", omega_mg=0.8)
    if cheb:
        kw.update(smoother="chebyshev", nu_pre=2, nu_post=2, weights="none", dt=0.001)
    g = w.Context(n, n, 1.0 / n, **kw)
    gl = g.layout
    U = g.zeros()
    its_g, lin_g, st_g = g.newton(U, rtol=1e-8, maxit=12)
    torch.cuda.synchronize()
    ref = _fields(U.cpu().numpy(), gl)
    g.close()
    assert st_g == "WRMG_OK"
    hub = w.LoopbackHub(P)

    def rank_fn(r):
        st = torch.cuda.Stream()
        with torch.cuda.stream(st):
            c = w.Context(n, n, 1.0 / n, rank=r, nranks=P, hub=hub, stream=st.cuda_stream, **kw)
            lay = c.layout
            u = c.zeros()
            its, lin, status = c.newton(u, rtol=1e-8, maxit=12)
            st.synchronize()
            res = {"its": its, "lin": lin, "st": status, "U": _owned(u.cpu().numpy(), lay)}
            c.close()
            return res

    outs = _run_ranks(P, rank_fn)
    hub.close()
    for o in outs:
        assert o["st"] == "WRMG_OK" and o["its"] == its_g and o["lin"] == lin_g, (o["its"], o["lin"], its_g, lin_g)
    e = _rel(_assemble(outs, "U", gl), ref)
    assert e <= 1e-8, f"U: rel {e:.3e}"


def test_ns_strip_canonical_fill_and_window():
    """bench.py's per-rank inputs of the NS strips: the R6 draws at global canonical
    ids (ns_fill_canonical) and the host window of a global vector (ns_window) equal
    the global vector's columns on every local column of every field."""
    import torch
    import paper_2407_13997_b200 as w
    import bench
    P, n, k, q, N = 2, 8, 2, 1, 2
    kw = dict(degree=k, q=q, nslabs=N, dt=0.1, ncoarse=2, problem="ns", reynolds=10.0, bc="lid")
    g = w.Context(n, n, 1.0 / n, **kw)
    gl = g.layout
    fg = bench.ns_fill_canonical(g, k, n).cpu().numpy()
    g.close()
    hub = w.LoopbackHub(P)

    def rank_fn(r):
        st = torch.cuda.Stream()
        with torch.cuda.stream(st):
            c = w.Context(n, n, 1.0 / n, rank=r, nranks=P, hub=hub, stream=st.cuda_stream, **kw)
            lay = c.layout
            fl = bench.ns_fill_canonical(c, k, n)
            st.synchronize()
            got = fl.cpu().numpy()
            win = bench.ns_window(fg, lay, gl["ly"], gl["lx"], gl["lpy"], gl["lpx"], gl["nt"])
            c.close()
            return got, _window(fg, gl, lay), win

    outs = _run_ranks(P, rank_fn)
    hub.close()
    for got, ref, win in outs:
        assert np.array_equal(got, ref) and np.array_equal(win, ref)
