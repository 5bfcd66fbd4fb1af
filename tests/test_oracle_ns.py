"""Oracle pins for the space-time Navier-Stokes discretisation (eq. nsfem,
PAPER.md:245-271) and its solver pieces (P17 and R17-R19, R22)."""
import numpy as np
import pytest

import wrmg_inputs as wi
from oracle import krylov, mesh, ns
from wrmg_testutil import read_golden


@pytest.mark.parametrize("k,q", [(1, 0), (1, 1), (2, 1)])
def test_P17_finite_difference_jacobian(k, q):
    """(F(U + eps d) - F(U)) / eps -> J(U) d with error O(eps)."""
    p = ns.NSProblem(mesh.unit_square(3), k, q, 3, 0.1, R=10.0)
    rng = np.random.default_rng(k + q)
    U, d = rng.standard_normal(p.ndof), rng.standard_normal(p.ndof)
    Jd = p.jacobian(U) @ d
    F0 = p.residual(U)
    errs = [np.linalg.norm((p.residual(U + e * d) - F0) / e - Jd) / np.linalg.norm(Jd) for e in (1e-5, 1e-6)]
    assert errs[1] <= 1e-5 and errs[1] < errs[0] * 0.2


def test_P17_reynolds_independent_at_zero_and_pressure_shift():
    p1 = ns.NSProblem(mesh.unit_square(3), 1, 1, 2, 0.1, R=1.0)
    p2 = ns.NSProblem(mesh.unit_square(3), 1, 1, 2, 0.1, R=100.0)
    Z = np.zeros(p1.ndof)
    assert abs(p1.jacobian(Z) - p2.jacobian(Z)).max() == 0.0
    # a constant pressure per (slab, temporal node) does not change the residual
    U = wi.spacetime_field(p1.ns, 2, 1, 3)
    U[p1.con_st] = p1.g_st[p1.con_st]
    V = p1.field_view(U).copy()
    V[2 * p1.Lu:, 1, 0] += 3.7
    assert np.allclose(p1.residual(V.reshape(-1)), p1.residual(U), atol=1e-12)


def test_divergence_blocks_are_transposes_and_vanish_on_solenoidal_fields():
    """R17: the (u,p) and (p,u) blocks are plain transposes; G^T I(w) -> 0 under
    refinement for the interpolant of a divergence-free field."""
    errs = []
    for n in (4, 8):
        p = ns.NSProblem(mesh.unit_square(n), 1, 0, 1, 0.1, R=1.0)
        Lu = p.Lu
        Gb = p.Gb.toarray()
        assert np.array_equal(Gb[:2 * Lu, 2 * Lu:], Gb[2 * Lu:, :2 * Lu].T)
        x, y = p.vel_xy[:, 0], p.vel_xy[:, 1]
        wx, wy = 2 * x ** 3 * y, -3 * x ** 2 * y ** 2  # curl of psi = x^3 y^2
        div = Gb[2 * Lu:, :Lu] @ wx + Gb[2 * Lu:, Lu:2 * Lu] @ wy
        errs.append(np.abs(div).max())
    assert errs[1] < errs[0] / 4


def test_vanka_star_patch_sizes_match_figure():
    """Interior Vanka+star patches: P2-P1 2*19 + 1 = 39; P3-P2 2*37 + 7 = 81, the
    37 velocity nodes and 7 pressure DoFs marked in Fig. patches (right)."""
    g = {r[0]: int(r[2]) for r in read_golden("patch_sizes.txt")}
    for k, size in ((1, 39), (2, 81)):
        p = ns.NSProblem(mesh.unit_square(6), k, 0, 1, 0.1, R=1.0)
        P, verts = ns.vanka_star_patches(p)
        # vertices whose closed star does not touch the (Dirichlet) boundary
        inner = [pt for pt, v in zip(P, verts) if 2 <= v % 7 <= 4 and 2 <= v // 7 <= 4]
        assert {pt.size for pt in inner} == {size}
        if k == 2:
            pt = inner[0]
            nvel = np.sum(pt < p.Lu)
            npre = np.sum(pt >= 2 * p.Lu)
            assert nvel == g["vanka_star_P3P2_velocity_nodes"] and npre == g["vanka_star_P3P2_pressure"]


def test_one_level_vcycle_is_exact_and_fgmres_converges():
    H = ns.NSHierarchy(4, 4, 0.25, 1, 1, 3, 0.1, R=100.0)
    p = H.fine
    b = wi.spacetime_field(p.ns, 3, 1, 0)
    b[p.con_st] = 0.0
    b = p.project_pressure(b)
    A = H.A[-1]
    z = ns.vcycle(H, b)
    assert np.linalg.norm(p.project_pressure(b - A @ z)) <= 1e-10 * np.linalg.norm(b)
    H2 = ns.NSHierarchy(8, 8, 0.125, 1, 1, 3, 0.1, R=100.0, omega_mg=0.8)
    p2 = H2.fine
    b2 = wi.spacetime_field(p2.ns, 3, 1, 0)
    b2[p2.con_st] = 0.0
    b2 = p2.project_pressure(b2)
    x, its, hist, st = krylov.fgmres(lambda v: H2.A[-1] @ v, lambda r: ns.vcycle(H2, r), b2, rtol=1e-8)
    assert st == "converged" and its < 40


def test_newton_cavity_converges_quadratically():
    """Newton-FGMRES-WRMG on a tiny lid-driven cavity:
    the nonlinear residual drops below 1e-8 of its initial value."""
    H = ns.NSHierarchy(4, 4, 0.25, 1, 0, 3, 0.02, R=10.0)
    U, hist, lin = ns.newton(H, rtol=1e-8, maxit=12)
    assert hist[-1] <= 1e-8 * hist[0]
    assert len(hist) <= 8


def test_ns_chebyshev_degree_one_is_damped_vanka():
    """Chebyshev with nu = 1 is one Vanka+star sweep damped
    by 1 / theta, theta = 0.65 lam, followed by the pressure projection (R19)."""
    from oracle import smoother
    H = ns.NSHierarchy(4, 4, 0.25, 1, 1, 2, 0.01, 10.0, bc="lid", smoother_kind="chebyshev", nu_pre=1,
                       nu_post=1, weight_mode="none", n_coarse=2, cheb_steps=12)
    l = len(H.probs) - 1
    p = H.probs[l]
    b = wi.spacetime_field(p.ns, 2, 1, 9)
    b[p.con_st] = 0.0
    x1 = ns.ns_chebyshev(H, l, np.zeros(p.ndof), b, 1)
    ref = p.project_pressure(smoother.wr_sweep(p, H.A[l], np.zeros(p.ndof), b, H.factors[l],
                                               1.0 / (0.65 * H.lam[l]), H.w[l]))
    assert np.allclose(x1, ref, rtol=1e-12, atol=1e-15)


def test_jacobian_residual_rows_equal_assembled_operator():
    """Row-by-row element evaluation of b - J(W) x (used for the full-size C3
    parity) equals the explicitly assembled space-time Jacobian."""
    p = ns.NSProblem(mesh.unit_square(4), 1, 1, 3, 0.1, R=50.0)
    W = 0.5 * wi.spacetime_field(p.ns, 3, 1, 4)
    x = wi.spacetime_field(p.ns, 3, 1, 5)
    b = wi.spacetime_field(p.ns, 3, 1, 6)
    ref = (b - p.jacobian(W) @ x).reshape(p.ns, 3, 2)
    rows = np.arange(p.ns)
    got = p.jacobian_residual_rows(rows, x, b, W)
    assert np.allclose(got, ref, rtol=1e-12, atol=1e-12 * np.abs(ref).max())


# ------------------------------------------------------------------ Chorin (N2)
def test_chorin_exact_solution_solves_the_momentum_equation():
    """PAPER.md:283-299 / R27: the exact Chorin velocity is solenoidal and, with the
    corrected pressure, solves u_t - Lap u + R (u.grad) u + grad p = 0 (central
    differences at random points); the printed pressure does not."""
    rng = np.random.default_rng(3)
    R, d = 10.0, 1e-4
    u = lambda x, y, t: np.array(wi.chorin_velocity(x, y, t))
    for x, y, t in rng.uniform(0.05, 0.95, size=(5, 3)) * [1, 1, 0.1]:
        ux, uy = (u(x + d, y, t) - u(x - d, y, t)) / (2 * d), (u(x, y + d, t) - u(x, y - d, t)) / (2 * d)
        ut = (u(x, y, t + d) - u(x, y, t - d)) / (2 * d)
        lap = (u(x + d, y, t) + u(x - d, y, t) + u(x, y + d, t) + u(x, y - d, t) - 4 * u(x, y, t)) / d ** 2
        u0 = u(x, y, t)
        conv = u0[0] * ux + u0[1] * uy
        for pf, ok in ((lambda X, Y: wi.chorin_pressure(X, Y, t, R), True),
                       (lambda X, Y: R * np.pi / 4 * (np.cos(2 * np.pi * X) + np.cos(2 * np.pi * Y))
                        * np.exp(-4 * np.pi ** 2 * t), False)):
            gp = np.array([(pf(x + d, y) - pf(x - d, y)) / (2 * d), (pf(x, y + d) - pf(x, y - d)) / (2 * d)])
            res = np.abs(ut - lap + R * conv + gp).max()
            assert (res < 1e-5) == ok, res
        assert abs(ux[0] + uy[1]) < 1e-8


def test_triangle_rule_integrates_monomials_exactly():
    from oracle import fem
    for npts in (2, 4, 6):
        xi, w = ns.triangle_rule(npts)
        for p in range(2 * npts - 1):
            for s in range(2 * npts - 1 - p):
                got = np.sum(w * xi[:, 0] ** p * xi[:, 1] ** s)
                assert abs(got - fem.mono_integral(p, s)) <= 1e-14 * max(1.0, fem.mono_integral(p, s)) + 1e-16


@pytest.mark.parametrize("k,q", [(1, 1), (2, 2)])
def test_velocity_l2_error_pins(k, q):
    """velocity_l2_error: zero for the interpolant of a field of
    degree <= k+1 in space and <= q in time; the closed form int_0^T int |u|^2 =
    T^3/27 for u = (x y t, 0) (needs k+1 >= 2, q >= 1); the closed form
    (1/2)(1 - exp(-4 pi^2 T)) / (4 pi^2) for U = 0 against the Chorin velocity."""
    n, N, T = 3, 2, 0.1
    p = ns.NSProblem(mesh.unit_square(n), k, q, N, T / N, 1.0, bc="dirichlet0")
    xy, tau = p.vel_xy, p.tm.nodes
    t = ((np.arange(N)[:, None] + tau[None, :]) * p.dt).ravel()
    f = lambda x, y, t: (x * y * t + (x ** (k + 1) - 2 * y) * t ** q, y ** (k + 1) * (1 + t ** q) - x * y)
    fx, fy = f(xy[:, 0:1], xy[:, 1:2], t[None, :])
    U = np.concatenate([fx, fy, np.zeros((p.Lp, t.size))]).ravel()
    assert ns.velocity_l2_error(p, U, f) < 1e-13
    g = lambda x, y, t: (x * y * t, 0.0 * x * y * t)
    gx, gy = g(xy[:, 0:1], xy[:, 1:2], t[None, :])
    U = np.concatenate([gx, gy, np.zeros((p.Lp, t.size))]).ravel()
    zero = lambda x, y, t: (0.0 * x * y * t, 0.0 * x * y * t)
    assert abs(ns.velocity_l2_error(p, U, zero) - np.sqrt(T ** 3 / 27)) < 1e-14
    ref = np.sqrt(0.5 * (1 - np.exp(-4 * np.pi ** 2 * T)) / (4 * np.pi ** 2))
    got = ns.velocity_l2_error(p, np.zeros(p.ndof), wi.chorin_velocity, nspace=10, ntime=10)
    assert abs(got - ref) < 1e-9 * ref


def test_chorin_newton_error_decreases_like_one_over_N():
    """Chorin problem (R28): Newton-FGMRES-WRMG with the exact
    velocity as Dirichlet data converges in a few steps and, at temporal degree 0,
    the space-time velocity error falls ~2x when N doubles (the 1/N column of
    Table tab:chorin:mg_errors)."""
    n, k, q, T, R = 4, 1, 0, 0.1, 10.0
    errs = []
    for N in (2, 4):
        H = ns.NSHierarchy(n, n, 1.0 / n, k, q, N, T / N, R, bc="dirichlet0", n_coarse=2)
        H.fine.set_boundary_data(wi.chorin_boundary_data(n, n, 1.0 / n, k, N, q, T / N))
        U, hist, lin = ns.newton(H, rtol=1e-8, maxit=10, u0=wi.chorin_u0(n, n, 1.0 / n, k))
        assert hist[-1] <= 1e-8 * hist[0] and len(lin) <= 6
        errs.append(ns.velocity_l2_error(H.fine, U, wi.chorin_velocity))
    assert 1.6 < errs[0] / errs[1] < 2.4, errs


@pytest.mark.parametrize("q", [0, 1, 2])
def test_chorin_boundary_data_interpolates_at_gauss_points(q):
    """R28: on every slab the temporal polynomial of the boundary data (R2 nodal
    basis, evaluated by the oracle's DG basis) equals the exact velocity at the
    q+1 Gauss-Legendre points."""
    from oracle import dg
    n, k, N, dt = 2, 1, 3, 0.05
    G = wi.chorin_boundary_data(n, n, 1.0 / n, k, N, q, dt)
    Lu = (2 * n + 1) ** 2
    V = G.reshape(-1, N, q + 1)
    g = 0.5 * (np.polynomial.legendre.leggauss(q + 1)[0] + 1.0)
    B = dg.TemporalMatrices(q, dt).eval(g)          # (q+1 points, q+1 basis)
    xy = mesh.node_coords(mesh.unit_square(n), k + 1)
    for nn in range(N):
        ex = wi.chorin_velocity(xy[:, 0:1], xy[:, 1:2], (nn + g[None, :]) * dt)
        assert np.allclose(V[:Lu, nn] @ B.T, ex[0], atol=1e-14)
        assert np.allclose(V[Lu:2 * Lu, nn] @ B.T, ex[1], atol=1e-14)
    assert not V[2 * Lu:].any()
