"""Round-2 oracle pins for the functions VERDICT r01 listed as open.

* ``smoother.weights`` / ``wr_sweep`` with mu > 1 (R11):
  with every patch solve replaced by the identity, one sweep from u = 0 is
  u = omega sum_p R_p^T W_p R_p b, i.e. omega * b on every covered free DoF when
  W = 1/mu (partition of unity), and omega * mu_i * b without weights, mu_i counted
  here from the patch lists.  A wrong 1/mu, a missed node or a doubled one fails.
* ``multigrid.chebyshev`` for nu >= 2: with a
  diagonal operator and B = I the error after nu steps is the classical Chebyshev
  factor T_nu((theta - t)/delta) / T_nu(theta/delta) times the initial error, with
  T_nu evaluated from its cos / cosh definition, not from the three-term recurrence
  the oracle uses.
* ``multigrid.estimate_lambda`` (R-cheb): with as many Arnoldi
  steps as the free subspace has dimensions the Ritz values are the eigenvalues of
  B A on that subspace -- compared with a dense eigen-solve of B A built column by
  column.  Plus SPEC.md:436: B = A^-1 (one patch holding every free DoF) gives 1.
* ``ns.eisenstat_walker``: a table of values
  worked out with 40-digit decimal arithmetic (tests/golden/eisenstat_walker.txt)
  and the defining properties of choice 2 (cap, safeguard, superlinear decay).
* ``ns.inject`` (R13): the coarse Taylor-Hood nodes are fine nodes, so the
  injected nodal interpolant of any function equals its coarse nodal interpolant.
"""
import math
import types

import numpy as np
import pytest
import scipy.sparse as sp

import wrmg_inputs as wi
from oracle import heat, multigrid, ns, patches, smoother
from oracle.mesh import Mesh
from wrmg_testutil import read_golden


# ------------------------------------------------------------ POU weights (R11)
@pytest.mark.parametrize("k,q", [(2, 1), (3, 0), (3, 1)])
@pytest.mark.parametrize("omega", [1.0, 0.7])
def test_pou_weights_identity_patch_solves(monkeypatch, k, q, omega):
    p = heat.unit_square_problem(4, k, q, 3, 0.1)
    b = p.rhs(wi.spacetime_field(p.nnode, 3, q, 2))
    P, _ = patches.vertex_star_patches(p.mesh, k, p.constrained)
    fac = smoother.PatchFactors(p, p.A, P)
    monkeypatch.setattr(smoother.PatchFactors, "solve", lambda self, pi, g: g.copy())
    mu = np.bincount(np.concatenate(P), minlength=p.nnode)  # patches containing each node
    assert mu.max() == k  # P2: 2, P3: 3 (edge / cell interiors shared by 2 / 3 vertex stars)
    free = np.repeat(p.free, p.NT)
    u = smoother.wr_sweep(p, p.A, np.zeros(p.ndof), b, fac, omega, smoother.weights(P, p.nnode, "pou"))
    assert np.allclose(u[free], omega * b[free], rtol=4e-16, atol=0)
    assert np.all(u[~free] == 0.0)
    u1 = smoother.wr_sweep(p, p.A, np.zeros(p.ndof), b, fac, omega, smoother.weights(P, p.nnode, "none"))
    assert np.allclose(u1, omega * np.repeat(mu, p.NT) * b, rtol=4e-16, atol=0)


# ------------------------------------------------------ Chebyshev nu >= 2 (N1)
def _cheb_T(nu, x):
    if abs(x) <= 1.0:
        return math.cos(nu * math.acos(x))
    s = 1.0 if x > 0 or nu % 2 == 0 else -1.0
    return s * math.cosh(nu * math.acosh(abs(x)))


@pytest.mark.parametrize("nu", [1, 2, 3, 4])
def test_chebyshev_error_factor_on_diagonal_model(monkeypatch, nu):
    lam = 2.0
    t = np.array([0.1, 0.3, 0.5, 0.8, 1.0, 1.3, 1.7, 2.0, 2.1, 2.6])  # eigenvalues of B A
    L = types.SimpleNamespace(prob=types.SimpleNamespace(A=sp.diags(t).tocsr()))
    monkeypatch.setattr(multigrid, "relaxation", lambda L_, r: r.copy())  # B = I
    xs = np.linspace(1.0, 2.0, t.size)
    b = t * xs
    u = multigrid.chebyshev(L, np.zeros_like(b), b, lam, nu)
    lo, hi = 0.25 * lam, 1.05 * lam
    theta, delta = 0.5 * (hi + lo), 0.5 * (hi - lo)
    fac = np.array([_cheb_T(nu, (theta - ti) / delta) / _cheb_T(nu, theta / delta) for ti in t])
    assert np.allclose(xs - u, fac * xs, rtol=1e-12, atol=1e-14)
    inside = (t >= lo) & (t <= hi)
    assert np.all(np.abs(fac[inside]) <= 1.0 / _cheb_T(nu, theta / delta) + 1e-14)


def test_chebyshev_identity_operator_sweep_interval():
    """op = identity, sweep = identity, interval [0.25, 1.05]: every error
    component is scaled by the degree-2 factor at 1, T_2((0.65 - 1)/0.4) / T_2(0.65/0.4)."""
    n = 6
    L = types.SimpleNamespace(prob=types.SimpleNamespace(A=sp.identity(n, format="csr")))
    orig = multigrid.relaxation
    try:
        multigrid.relaxation = lambda L_, r: r.copy()
        e0 = np.linspace(-1.0, 2.0, n)
        u = multigrid.chebyshev(L, -e0, np.zeros(n), 1.0, 2)  # x* = 0, so e = -u
    finally:
        multigrid.relaxation = orig
    x, y = -0.35 / 0.4, 0.65 / 0.4
    f = (2 * x * x - 1) / (2 * y * y - 1)
    assert np.allclose(-u, f * e0, rtol=1e-13, atol=1e-15)


# ------------------------------------------------------ lambda estimate (R-cheb)
def test_estimate_lambda_equals_dense_spectrum():
    p = heat.unit_square_problem(2, 2, 1, 2, 0.1)
    L = multigrid.Level(p, "pou")
    free = np.nonzero(np.repeat(p.free, p.NT))[0]
    nf = free.size
    BA = np.zeros((nf, nf))
    for c, j in enumerate(free):
        e = np.zeros(p.ndof)
        e[j] = 1.0
        BA[:, c] = multigrid.relaxation(L, p.A @ e)[free]
    exact = np.abs(np.linalg.eigvals(BA)).max()
    with np.errstate(divide="ignore", invalid="ignore"):
        est = multigrid.estimate_lambda(L, steps=nf, seed=7)
    assert est == pytest.approx(exact, rel=1e-8)


def test_estimate_lambda_exact_preconditioner_is_one():
    """B = A^-1 (a single patch of all free DoFs, unit weights) -> lambda = 1."""
    p = heat.unit_square_problem(3, 1, 0, 3, 0.1)
    L = multigrid.Level(p, "none")
    allfree = [np.nonzero(p.free)[0]]
    L.patches = allfree
    L.w = np.ones(p.nnode)
    L.factors = smoother.PatchFactors(p, p.A, allfree)
    with np.errstate(divide="ignore", invalid="ignore"):
        est = multigrid.estimate_lambda(L, steps=3, seed=7)
    assert est == pytest.approx(1.0, abs=1e-10)


# ------------------------------------------------------ Eisenstat-Walker (R22)
def test_eisenstat_walker_table():
    for row in read_golden("eisenstat_walker.txt"):
        eta_prev, ratio, want = float(row[0]), float(row[1]), float(row[2])
        got = ns.eisenstat_walker(eta_prev, ratio, 1.0)
        assert got == pytest.approx(want, rel=1e-13), row


def test_eisenstat_walker_properties():
    a = (1 + 5 ** 0.5) / 2
    rng = np.random.default_rng(3)
    for _ in range(200):
        eta_prev = rng.uniform(1e-6, 0.9)
        fprev = rng.uniform(0.1, 10.0)
        fn = fprev * rng.uniform(1e-6, 2.0)
        eta = ns.eisenstat_walker(eta_prev, fn, fprev)
        assert 0.0 < eta <= 0.9
        if eta_prev ** a > 0.1:
            assert eta >= min(eta_prev ** a, 0.9) * (1 - 1e-15)
        if eta < 0.9 and eta_prev ** a <= 0.1:
            assert eta == pytest.approx((fn / fprev) ** a, rel=1e-14)
    # superlinear decay: a quadratically converging residual sequence drives eta to 0
    eta, f = 0.3, [1.0, 1e-1, 1e-3, 1e-7]
    for k2 in range(1, len(f)):
        eta = ns.eisenstat_walker(eta, f[k2], f[k2 - 1])
    assert eta < 1e-6


# ------------------------------------------------------------------ inject (R13)
@pytest.mark.parametrize("k,q", [(1, 1), (2, 0)])
def test_inject_is_nodal_sampling(k, q):
    N, dt = 3, 0.2
    fine = ns.NSProblem(Mesh(4, 4, 0.25), k, q, N, dt, R=10.0)
    coarse = ns.NSProblem(Mesh(2, 2, 0.5), k, q, N, dt, R=10.0)
    tn = lambda n, a: (n + (a / q if q else 0.5)) * dt
    fu = lambda x, y, t: np.sin(3 * x + 2 * y + t) + x * y
    fv = lambda x, y, t: np.cos(x - 4 * y * t) - y
    fp = lambda x, y, t: np.exp(x * y) + t

    def interp(prob):
        V = np.zeros((prob.ns, N, q + 1))
        for n in range(N):
            for a in range(q + 1):
                t = tn(n, a)
                V[:prob.Lu, n, a] = fu(prob.vel_xy[:, 0], prob.vel_xy[:, 1], t)
                V[prob.Lu:2 * prob.Lu, n, a] = fv(prob.vel_xy[:, 0], prob.vel_xy[:, 1], t)
                V[2 * prob.Lu:, n, a] = fp(prob.p_xy[:, 0], prob.p_xy[:, 1], t)
        return V.reshape(-1)

    got = ns.inject(fine, coarse, interp(fine))
    assert np.array_equal(got, interp(coarse))
