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
