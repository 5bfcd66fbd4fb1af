"""Slab windows of the Navier-Stokes Vanka inverses: a level whose
stored inverses do not fit keeps W slabs and recomputes them in every sweep, the
jump carried across windows in a per-patch buffer.  The result must be the stored
form's: GPU = oracle (R23, 1e-10) on ragged windows, identical Krylov and Newton
counts, for the staged (m = 78) and the chunked-ring (m = 162, C4's P3-P2) sweeps."""
import numpy as np
import pytest

import wrmg_inputs as wi
from test_gpu_ns import _dev, _host, _rhs, assert_parity

pytestmark = pytest.mark.gpu


def _ctx(n, k, q, N, dt, R=100.0, wind=True):
    import paper_2407_13997_b200 as w
    c = w.Context(n, n, 1.0 / n, degree=k, q=q, nslabs=N, dt=dt, problem="ns", reynolds=R, bc="lid",
                  omega_mg=0.8)
    W = wi.wind_state(n, n, 1.0 / n, k, N, q, dt) if wind else None
    if W is not None:
        c.linearize(_dev(W))
    return c, W


@pytest.mark.parametrize("k,N,win", [(1, 5, 2), (2, 4, 3), (1, 6, 1)])
def test_windowed_sweeps_match_oracle(monkeypatch, k, N, win):
    from oracle import ns, smoother
    monkeypatch.setenv("WRMG_NS_WINDOW", str(win))
    dt = 1.0 / N
    c, W = _ctx(8, k, 1, N, dt)
    H = ns.NSHierarchy(8, 8, 1.0 / 8, k, 1, N, dt, 100.0, W=W, bc="lid", omega_mg=0.8)
    p = H.fine
    b, bref = _rhs(c, p)
    u = c.zeros()
    uref = np.zeros(p.ndof)
    for it in range(3):
        c.smooth(u, b, 1, 0.8)
        uref = p.project_pressure(smoother.wr_sweep(p, H.A[-1], uref, bref, H.factors[-1], 0.8, H.w[-1]))
        assert_parity(_host(u), uref, what=f"windowed sweep {it}")
    c.close()


def test_windowed_vcycle_and_fgmres_match_oracle(monkeypatch):
    from oracle import krylov, ns
    monkeypatch.setenv("WRMG_NS_WINDOW", "3")
    n, k, N, R = 16, 1, 7, 10.0
    dt = 1.0 / N
    c, W = _ctx(n, k, 1, N, dt, R=R)
    H = ns.NSHierarchy(n, n, 1.0 / n, k, 1, N, dt, R, W=W, bc="lid", omega_mg=0.8)
    p = H.fine
    b, bref = _rhs(c, p, seed=3)
    z = c.empty()
    c.vcycle(b, z)
    assert_parity(_host(z), ns.vcycle(H, bref), what="windowed V(1,1)")
    x = c.empty()
    its, rel, st = c.fgmres(b, x, restart=30, maxit=200, rtol=1e-8)
    xref, its_ref, hist, st_ref = krylov.fgmres(lambda v: H.A[-1] @ v, lambda r: ns.vcycle(H, r), bref,
                                                restart=30, maxit=200, rtol=1e-8)
    assert st == "WRMG_OK" and st_ref == "converged" and its == its_ref
    assert_parity(_host(x), xref, tol=1e-9, what="windowed FGMRES iterate")
    c.close()


def test_windowed_newton_cavity_p3p2(monkeypatch):
    """C4's pair (P3-P2 x DG1, m = 162: chunked-ring sweep) with 2-slab windows."""
    from oracle import ns
    import paper_2407_13997_b200 as w
    monkeypatch.setenv("WRMG_NS_WINDOW", "2")
    n, k, q, N, dt, R = 8, 2, 1, 3, 0.05, 10.0
    c = w.Context(n, n, 1.0 / n, degree=k, q=q, nslabs=N, dt=dt, problem="ns", reynolds=R, bc="lid",
                  omega_mg=0.8)
    H = ns.NSHierarchy(n, n, 1.0 / n, k, q, N, dt, R, bc="lid", omega_mg=0.8)
    Uref, hist, lin = ns.newton(H, rtol=1e-8, maxit=12)
    U = c.zeros()
    its, lin_its, st = c.newton(U, rtol=1e-8, maxit=12)
    assert st == "WRMG_OK" and its == len(lin) and lin_its == sum(lin)
    assert_parity(_host(U), Uref, tol=1e-8, what="windowed Newton solution")
    c.close()


def test_budget_windows_match_stored(monkeypatch):
    """A store budget below the inverses' size halves the largest level's window until
    it fits; the sweeps then equal the stored form's (to the atomic order, 1e-12)."""
    n, k, N = 16, 1, 8
    dt = 1.0 / N
    c0, W = _ctx(n, k, 1, N, dt)
    per_slab = (16 - 1) ** 2 * (2 * 39) ** 2 * 8.0  # finest level, one slab
    monkeypatch.setenv("WRMG_NS_STORE_GB", str(3.0 * per_slab / 1e9))
    c1, _ = _ctx(n, k, 1, N, dt)
    from oracle import ns
    p = ns.NSHierarchy(n, n, 1.0 / n, k, 1, N, dt, 100.0, W=None, bc="lid", omega_mg=0.8).fine
    b0, _ = _rhs(c0, p, seed=5)
    b1, _ = _rhs(c1, p, seed=5)
    u0, u1 = c0.zeros(), c1.zeros()
    c0.smooth(u0, b0, 2, 0.8)
    c1.smooth(u1, b1, 2, 0.8)
    assert_parity(_host(u1), _host(u0), tol=1e-12, what="budget windows vs stored")
    z0, z1 = c0.empty(), c1.empty()
    c0.vcycle(b0, z0)
    c1.vcycle(b1, z1)
    assert_parity(_host(z1), _host(z0), tol=1e-12, what="budget windows V(1,1)")
    c0.close()
    c1.close()
