"""GPU parity of the Navier-Stokes path (Taylor-Hood x DG(q), Newton Jacobian at
the C3 wind, Vanka+star WR smoother, V-cycle, FGMRES, Newton) against the oracle
(oracle/ns.py) on the same seeded inputs.  Tolerance: DESIGN.md R23 (1e-10
relative per vector, identical Krylov / Newton iteration counts)."""
import numpy as np
import pytest

import wrmg_inputs as wi

pytestmark = pytest.mark.gpu

TOL = 1e-10


def _torch():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    return torch


def _dev(x):
    torch = _torch()
    return torch.as_tensor(np.ascontiguousarray(x), dtype=torch.float64, device="cuda:0")


def _host(t):
    _torch().cuda.synchronize()
    return t.detach().cpu().numpy()


def assert_parity(gpu, ref, tol=TOL, what=""):
    gpu, ref = np.asarray(gpu), np.asarray(ref)
    e2 = np.linalg.norm(gpu - ref) / np.linalg.norm(ref)
    einf = np.max(np.abs(gpu - ref)) / np.max(np.abs(ref))
    assert e2 <= tol and einf <= tol, f"{what}: rel2 {e2:.3e} relinf {einf:.3e}"
    return e2, einf


def _setup(n, k, q, N, R=100.0, omega_mg=0.8, bc="lid", wind=True, T=1.0):
    """GPU context and oracle hierarchy linearised at the C3 wind (R18)."""
    import paper_2407_13997_b200 as w
    from oracle import ns
    dt = T / N
    W = wi.wind_state(n, n, 1.0 / n, k, N, q, dt) if wind else None
    c = w.Context(n, n, 1.0 / n, degree=k, q=q, nslabs=N, dt=dt, problem="ns", reynolds=R, bc=bc,
                  omega_mg=omega_mg)
    if W is not None:
        c.linearize(_dev(W))
    H = ns.NSHierarchy(n, n, 1.0 / n, k, q, N, dt, R, W=W, bc=bc, omega_mg=omega_mg)
    return c, H, W


def _rhs(c, p, seed=0):
    """b of config C3 (R6): U[-1,1) on free rows, 0 on constrained, pressure projected."""
    f = wi.spacetime_field(p.ns, p.N, p.q, seed)
    b = c.empty()
    c.rhs(_dev(f), b)
    bref = f.copy()
    bref[p.con_st] = 0.0
    return b, p.project_pressure(bref)


@pytest.mark.parametrize("k,q,N", [(1, 1, 3), (2, 1, 2), (1, 0, 4), (1, 2, 2)])
def test_ns_apply_matches_jacobian(k, q, N):
    c, H, W = _setup(8, k, q, N)
    p = H.fine
    x = wi.spacetime_field(p.ns, N, q, 7)
    y = c.empty()
    c.apply(_dev(x), y)
    assert_parity(_host(y), H.A[-1] @ x, what="J x")
    b = wi.spacetime_field(p.ns, N, q, 8)
    r = c.empty()
    c.residual(_dev(x), _dev(b), r)
    assert_parity(_host(r), b - H.A[-1] @ x, what="b - J x")
    c.close()


@pytest.mark.parametrize("k", [1, 2])
def test_ns_nonlinear_residual(k):
    c, H, W = _setup(8, k, 1, 3, wind=False)
    p = H.fine
    U = 0.3 * wi.spacetime_field(p.ns, 3, 1, 11)
    b = np.zeros(p.ndof)
    b[p.con_st] = p.g_st[p.con_st]
    r = c.empty()
    c.residual(_dev(U), _dev(b), r, nonlinear=True)
    assert_parity(_host(r), -p.residual(U), what="-F(U)")
    c.close()


@pytest.mark.parametrize("k,omega", [(1, 1.0), (2, 0.8)])
def test_ns_smoother_sweeps(k, omega):
    from oracle import smoother
    c, H, W = _setup(8, k, 1, 3)
    p = H.fine
    b, bref = _rhs(c, p)
    assert_parity(_host(b), bref, what="rhs")
    u = c.zeros()
    uref = np.zeros(p.ndof)
    for it in range(3):
        c.smooth(u, b, 1, omega)
        uref = p.project_pressure(smoother.wr_sweep(p, H.A[-1], uref, bref, H.factors[-1], omega, H.w[-1]))
        assert_parity(_host(u), uref, what=f"sweep {it}")
    c.close()


@pytest.mark.parametrize("n,k,N", [(8, 1, 3), (16, 1, 3), (8, 2, 3), (8, 1, 70)])
def test_ns_vcycle(n, k, N):
    from oracle import ns
    c, H, W = _setup(n, k, 1, N, T=0.02 * N / 64)
    p = H.fine
    b, bref = _rhs(c, p, seed=3)
    z = c.empty()
    c.vcycle(b, z)
    assert_parity(_host(z), ns.vcycle(H, bref), what="V(1,1)")
    c.close()


@pytest.mark.parametrize("n,k,q,N", [(4, 1, 1, 3), (4, 2, 1, 3), (4, 2, 0, 5), (2, 1, 0, 3)])
def test_ns_one_level_vcycle_is_pinned_coarse_solve(n, k, q, N):
    """Coarse slab blocks of m = 27 (CTA LU) and 246 / 323 / 646 (blocked
    Gauss-Jordan, kernels_gj.cu)."""
    from oracle import ns
    c, H, W = _setup(n, k, q, N)
    p = H.fine
    b, bref = _rhs(c, p, seed=4)
    z = c.empty()
    c.vcycle(b, z)
    zref = ns.vcycle(H, bref)
    assert_parity(_host(z), zref, what="coarse solve")
    assert np.linalg.norm(p.project_pressure(bref - H.A[-1] @ zref)) <= 1e-10 * np.linalg.norm(bref)
    c.close()


@pytest.mark.parametrize("n,k,N,R,T", [(8, 1, 4, 10.0, 1.0), (16, 1, 4, 20.0, 1.0), (8, 2, 3, 20.0, 1.0),
                                       (16, 1, 40, 10.0, 0.02 * 40 / 64)])
def test_ns_fgmres_iteration_count(n, k, N, R, T):
    """Cell Reynolds numbers R |w| h <= 6 (C3 itself: 100 * 4.7 / 64 = 7.4); at
    R |w| h ~ 30 the additive Vanka V(1,1) no longer contracts (oracle and GPU
    alike), so no iteration count would be compared."""
    from oracle import krylov, ns
    c, H, W = _setup(n, k, 1, N, R=R, T=T)
    p = H.fine
    b, bref = _rhs(c, p, seed=0)
    x = c.empty()
    its, rel, st = c.fgmres(b, x, restart=30, maxit=200, rtol=1e-8)
    xref, its_ref, hist, st_ref = krylov.fgmres(lambda v: H.A[-1] @ v, lambda r: ns.vcycle(H, r), bref,
                                                restart=30, maxit=200, rtol=1e-8)
    assert st == "WRMG_OK" and st_ref == "converged"
    assert its == its_ref
    assert_parity(_host(x), xref, tol=1e-9, what="FGMRES iterate")
    c.close()


@pytest.mark.parametrize("k", [1, 2])
def test_ns_newton_cavity(k):
    """Newton-FGMRES-WRMG (R22) on a small lid-driven cavity,
    P2-P1 and P3-P2 (C4's pair) x DG1: identical Newton and linear iteration
    counts, solution within 1e-8."""
    from oracle import ns
    n, q, N, dt, R = 8, 1, 3, 0.05, 10.0
    import paper_2407_13997_b200 as w
    c = w.Context(n, n, 1.0 / n, degree=k, q=q, nslabs=N, dt=dt, problem="ns", reynolds=R, bc="lid",
                  omega_mg=0.8)
    H = ns.NSHierarchy(n, n, 1.0 / n, k, q, N, dt, R, bc="lid", omega_mg=0.8)
    Uref, hist, lin = ns.newton(H, rtol=1e-8, maxit=12)
    U = c.zeros()
    its, lin_its, st = c.newton(U, rtol=1e-8, maxit=12)
    assert st == "WRMG_OK"
    assert its == len(lin) and lin_its == sum(lin)
    assert_parity(_host(U), Uref, tol=1e-8, what="Newton solution")
    c.close()


def test_ns_chebyshev_vcycle_and_newton():
    """Chebyshev-accelerated V(2,2) on the Vanka+star smoother (PAPER.md:366-379,
    R-cheb; unweighted patches) for the lid-driven cavity: lambda per level
    (re-estimated at every linearisation), one cycle, and Newton-FGMRES-WRMG
    with identical Newton and linear counts."""
    import paper_2407_13997_b200 as w
    from oracle import ns
    n, k, q, N, dt, R = 8, 1, 1, 4, 0.001, 10.0
    kw = dict(bc="lid")
    c = w.Context(n, n, 1.0 / n, degree=k, q=q, nslabs=N, dt=dt, problem="ns", reynolds=R, weights="none",
                  nu_pre=2, nu_post=2, smoother="chebyshev", **kw)
    H = ns.NSHierarchy(n, n, 1.0 / n, k, q, N, dt, R, smoother_kind="chebyshev", nu_pre=2, nu_post=2,
                       weight_mode="none", **kw)
    for l in range(1, len(H.probs)):
        assert abs(c.cheb_lambda(l) - H.lam[l]) <= 1e-10 * H.lam[l]
    p = H.fine
    f = wi.spacetime_field(p.ns, N, q, 5)
    b = c.empty()
    c.rhs(_dev(f), b)
    bref = f.copy()
    bref[p.con_st] = 0.0
    bref = p.project_pressure(bref)
    z = c.empty()
    c.vcycle(b, z)
    assert_parity(_host(z), ns.vcycle(H, bref), what="Chebyshev V(2,2)")
    Uref, hist, lin = ns.newton(H, rtol=1e-8, maxit=12)
    U = c.zeros()
    its, lin_its, st = c.newton(U, rtol=1e-8, maxit=12)
    assert st == "WRMG_OK" and its == len(lin) and lin_its == sum(lin)
    assert_parity(_host(U), Uref, tol=1e-8, what="Newton solution")
    c.close()


def test_ns_newton_with_initial_state():
    """Newton with the initial-state term (R7; wrmg_rhs_initial + wrmg_newton_rhs):
    one slab started from a nonzero velocity, as one step of the timestepping
    comparison; counts and solution equal the oracle's."""
    import paper_2407_13997_b200 as w
    from oracle import ns
    n, k, q, N, dt, R = 8, 1, 0, 1, 0.001, 10.0
    c = w.Context(n, n, 1.0 / n, degree=k, q=q, nslabs=N, dt=dt, problem="ns", reynolds=R, bc="lid",
                  weights="none", nu_pre=2, nu_post=2, smoother="chebyshev")
    H = ns.NSHierarchy(n, n, 1.0 / n, k, q, N, dt, R, bc="lid", smoother_kind="chebyshev", nu_pre=2, nu_post=2,
                       weight_mode="none")
    p = H.fine
    u0 = np.zeros(p.ns)
    x, y = p.vel_xy[:, 0], p.vel_xy[:, 1]
    u0[:p.Lu] = np.sin(np.pi * x) * np.sin(np.pi * y) ** 2
    u0[p.Lu:2 * p.Lu] = -np.sin(np.pi * x) ** 2 * np.sin(np.pi * y)
    Uref, hist, lin = ns.newton(H, rtol=1e-8, maxit=12, u0=u0)
    rhs = c.zeros()
    c.rhs_initial(_dev(u0), rhs)
    U = c.zeros()
    its, lin_its, st = c.newton(U, rtol=1e-8, maxit=12, rhs=rhs)
    assert st == "WRMG_OK" and its == len(lin) and lin_its == sum(lin)
    assert_parity(_host(U), Uref, tol=1e-8, what="Newton with u0")
    c.close()


def test_C3_fullsize_sampled_jacobian_rows():
    """C3 at its full size (BASELINE configs[2]: 64x64 P2-P1 x DG1, N = 64, Re = 100,
    Newton Jacobian at the wind, lid): b - J x from the GPU residual kernel, in the
    bench's launch configuration, against the oracle's row-by-row element
    evaluation on sampled velocity and pressure rows (every slab and temporal node)."""
    import paper_2407_13997_b200 as w
    from oracle import mesh as omesh
    from oracle import ns
    n, k, q, N, R = 64, 1, 1, 64, 100.0
    dt = 1.0 / N
    W = wi.wind_state(n, n, 1.0 / n, k, N, q, dt)
    c = w.Context(n, n, 1.0 / n, degree=k, q=q, nslabs=N, dt=dt, problem="ns", reynolds=R, bc="lid",
                  omega_mg=0.8)
    c.linearize(_dev(W))
    p = ns.NSProblem(omesh.unit_square(n), k, q, N, dt, R, bc="lid")
    x = wi.spacetime_field(p.ns, N, q, 21)
    b = wi.spacetime_field(p.ns, N, q, 22)
    r = c.empty()
    c.residual(_dev(x), _dev(b), r)
    got = _host(r).reshape(p.ns, N, q + 1)
    rng = np.random.default_rng(0)
    Lu, Lux = p.Lu, 2 * n + 1
    picks = [Lux + 1, 2 * Lux + 2, (Lux // 2) * Lux + Lux // 2, Lu - Lux - 2, Lu + Lux + 1, Lu + 3 * Lux + 5,
             2 * Lu, 2 * Lu + 66, 2 * Lu + p.Lp - 1]
    picks += list(rng.integers(0, p.ns, 20))
    ref = p.jacobian_residual_rows(picks, x, b, W)
    for ir, s_ in enumerate(picks):
        e = np.max(np.abs(got[s_] - ref[ir])) / max(np.max(np.abs(ref[ir])), 1e-300)
        assert e <= 1e-10, (s_, e)
    c.close()
