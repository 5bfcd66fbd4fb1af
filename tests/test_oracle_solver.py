"""Oracle pins P7-P10, P12, P15, P16, P18 (patches, smoother, transfers,
multigrid, FGMRES).  Each is checked against something other than the oracle's
own formula: dense/sparse direct solves, hand closed forms, polynomial
reproduction, textbook Krylov facts, the paper's Fig. patches."""
import numpy as np
import pytest
import scipy.sparse as sp
import scipy.sparse.linalg as spla

import wrmg_inputs as wi
from oracle import heat, krylov, mesh, multigrid, patches, smoother, transfer
from wrmg_testutil import read_golden


def _interior_patch_sizes(n, k):
    p = heat.unit_square_problem(n, k, 0, 1, 1.0, build_matrix=False)
    P, verts = patches.vertex_star_patches(p.mesh, k, p.constrained)
    sizes = {}
    for pt, v in zip(P, verts):
        I, J = v % (n + 1), v // (n + 1)
        if 1 <= I < n and 1 <= J < n:
            sizes.setdefault(pt.size, 0)
            sizes[pt.size] += 1
    return sizes, P, verts, p


@pytest.mark.parametrize("k,m_p,mu_max", [(1, 1, 1), (2, 7, 2), (3, 19, 3)])
def test_P10_vertex_star_patches(k, m_p, mu_max):
    n = 5
    sizes, P, verts, p = _interior_patch_sizes(n, k)
    assert list(sizes) == [m_p]
    mu = patches.multiplicity(P, p.nnode)
    assert mu.max() == mu_max
    assert np.all(mu[p.free] >= 1) and np.all(mu[p.constrained] == 0)  # cover; Dirichlet excluded
    # colouring (I - J) mod 3 of the patch vertex is conflict-free
    for c in range(3):
        sel = [pt for pt, v in zip(P, verts) if ((v % (n + 1)) - (v // (n + 1))) % 3 == c]
        allnodes = np.concatenate(sel)
        assert np.unique(allnodes).size == allnodes.size


def test_P10_figure_patch_size():
    rows = {r[0]: int(r[2]) for r in read_golden("patch_sizes.txt")}
    sizes, *_ = _interior_patch_sizes(4, 2)
    assert list(sizes) == [rows["vertex_star_P2"]]


def _small_problem(n=4, k=2, q=1, N=3, dt=0.1, kappa=1.0, seed=0):
    p = heat.unit_square_problem(n, k, q, N, dt, kappa=kappa)
    b = p.rhs(wi.spacetime_field(p.nnode, N, q, seed))
    return p, b


def test_P7_patch_march_equals_dense_solve():
    p, b = _small_problem()
    P, _ = patches.vertex_star_patches(p.mesh, p.k, p.constrained)
    fac = smoother.PatchFactors(p, p.A, P)
    rng = np.random.default_rng(1)
    for pi in (0, len(P) // 2, len(P) - 1):
        I = fac.I[pi]
        g = rng.standard_normal(I.size)
        Ap = p.A[I][:, I].toarray()
        assert np.allclose(fac.solve(pi, g), np.linalg.solve(Ap, g), rtol=1e-11, atol=1e-12)


def test_patch_blocks_kron_equal_restriction():
    """The Kronecker-built patch blocks used at full size equal A[I_p][:, I_p]."""
    for k, q in ((2, 1), (3, 2), (1, 0)):
        p, b = _small_problem(n=4, k=k, q=q, N=3)
        P, _ = patches.vertex_star_patches(p.mesh, k, p.constrained)
        for pt in (P[0], P[len(P) // 2], P[-1]):
            D, L = smoother.patch_blocks_kron(p, pt)
            I1, I0 = p.slab_indices(pt, 1), p.slab_indices(pt, 0)
            assert np.allclose(D, p.A[I1][:, I1].toarray(), rtol=0, atol=1e-15)
            assert np.allclose(L, p.A[I1][:, I0].toarray(), rtol=0, atol=1e-15)
            g = np.random.default_rng(0).standard_normal(pt.size * (q + 1) * p.N)
            fac = smoother.PatchFactors(p, p.A, [pt])
            assert np.allclose(smoother.patch_solve_kron(p, pt, g), fac.solve(0, g), rtol=1e-12, atol=1e-14)


@pytest.mark.parametrize("k,q", [(1, 0), (2, 1), (3, 1)])
def test_P8_single_patch_is_direct_solve(k, q):
    p, b = _small_problem(n=3, k=k, q=q)
    allfree = [np.nonzero(p.free)[0]]
    fac = smoother.PatchFactors(p, p.A, allfree)
    u = smoother.wr_sweep(p, p.A, np.zeros(p.ndof), b, fac, 1.0, np.ones(p.nnode))
    x = spla.spsolve(p.A.tocsc(), b)
    assert np.allclose(u, x, rtol=1e-10, atol=1e-13)


def test_P9_p1_dg0_closed_form_sweep():
    """C1 shape: P1 patches are single DoFs, x_n = (r_n + m_ii x_{n-1}) / (m_ii + dt k_ii),
    m_ii = h^2/2 = 1/512, k_ii = 4, dt = 1/16 -> denominator 0.251953125."""
    n, N = 16, 16
    p = heat.unit_square_problem(n, 1, 0, N, 1.0 / N)
    b = p.rhs(wi.spacetime_field(p.nnode, N, 0, 0))
    P, _ = patches.vertex_star_patches(p.mesh, 1, p.constrained)
    fac = smoother.PatchFactors(p, p.A, P)
    w = smoother.weights(P, p.nnode)
    assert np.all(w[p.free] == 1.0)
    u = smoother.wr_sweep(p, p.A, np.zeros(p.ndof), b, fac, 1.0, w).reshape(p.nnode, N)
    r = b.reshape(p.nnode, N)
    for i in np.nonzero(p.free)[0][::7]:
        x = 0.0
        for s in range(N):
            x = (r[i, s] + x / 512.0) / 0.251953125
            assert u[i, s] == pytest.approx(x, rel=1e-12)


def test_P18_order_independence():
    p, b = _small_problem(k=3)
    P, _ = patches.vertex_star_patches(p.mesh, p.k, p.constrained)
    fac = smoother.PatchFactors(p, p.A, P)
    w = smoother.weights(P, p.nnode)
    u0 = wi.spacetime_field(p.nnode, p.N, p.q, 7) * ~p.con_st
    a = smoother.wr_sweep(p, p.A, u0, b, fac, 0.8, w)
    order = np.random.default_rng(5).permutation(len(P))
    c = smoother.wr_sweep(p, p.A, u0, b, fac, 0.8, w, order=order)
    assert np.max(np.abs(a - c)) <= 1e-13 * np.max(np.abs(a))
    assert np.all(a[p.con_st] == u0[p.con_st])  # no correction on Dirichlet DoFs


@pytest.mark.parametrize("k", [1, 2, 3])
def test_P12_interpolation(k):
    c, f = mesh.Mesh(3, 2, 0.5), mesh.Mesh(6, 4, 0.25)
    P = transfer.interpolation(c, f, k)
    assert np.allclose(np.asarray(P.sum(axis=1)).ravel(), 1.0, atol=1e-13)
    # reproduces coarse polynomials of degree <= k exactly
    cxy, fxy = mesh.node_coords(c, k), mesh.node_coords(f, k)
    rng = np.random.default_rng(k)
    coef = rng.standard_normal((k + 1, k + 1))
    poly = lambda xy: sum(coef[i, j] * xy[:, 0] ** i * xy[:, 1] ** j
                          for i in range(k + 1) for j in range(k + 1 - i))
    assert np.allclose(P @ poly(cxy), poly(fxy), atol=1e-12)
    # fine nodes at coarse node positions carry a single entry 1
    cidx = mesh.node_index_from_coords(f, k, cxy)
    Pc = P[cidx].toarray()
    assert np.allclose(Pc, np.eye(cxy.shape[0]), atol=1e-14)


def test_P15_multigrid_sanity():
    # one-level hierarchy: V-cycle = exact solve
    H1 = multigrid.Hierarchy(4, 4, 0.25, 2, 1, 3, 0.1)
    assert len(H1.levels) == 1
    b = H1.fine.rhs(wi.spacetime_field(H1.fine.nnode, 3, 1, 0))
    assert np.allclose(multigrid.vcycle(H1, b), spla.spsolve(H1.fine.A.tocsc(), b), rtol=1e-10, atol=1e-14)
    # b = 0 gives z = 0; a V(1,1) cycle on C1's shape contracts
    H = multigrid.Hierarchy(16, 16, 1.0 / 16, 1, 0, 16, 1.0 / 16)
    p = H.fine
    assert np.all(multigrid.vcycle(H, np.zeros(p.ndof)) == 0.0)
    e = wi.spacetime_field(p.nnode, 16, 0, 4) * ~p.con_st
    for _ in range(3):
        e_new = e - multigrid.vcycle(H, p.A @ e)
        ratio = np.linalg.norm(e_new) / np.linalg.norm(e)
        assert ratio < 1.0
        e = e_new


def test_P16_fgmres_textbook():
    b = np.array([0.3, -1.2, 2.0])
    x, its, hist, st = krylov.fgmres(lambda v: v, lambda v: v, b)
    assert its == 1 and st == "converged" and np.allclose(x, b)
    D = np.array([1.0, 10.0])
    x, its, hist, st = krylov.fgmres(lambda v: D * v, lambda v: v, np.ones(2), rtol=1e-14)
    assert its <= 2 and np.allclose(x, [1.0, 0.1], rtol=1e-13)
    p, b = _small_problem(n=3, k=2)
    Ainv = lambda r: spla.spsolve(p.A.tocsc(), r)
    x, its, hist, st = krylov.fgmres(lambda v: p.A @ v, Ainv, b)
    assert its == 1
    H = multigrid.Hierarchy(8, 8, 1.0 / 8, 2, 1, 4, 0.25)
    b = H.fine.rhs(wi.spacetime_field(H.fine.nnode, 4, 1, 0))
    x, its, hist, st = krylov.fgmres(lambda v: H.fine.A @ v, lambda r: multigrid.vcycle(H, r), b)
    assert st == "converged"
    assert np.all(np.diff(hist) <= 1e-15 * hist[0])
    assert np.linalg.norm(b - H.fine.A @ x) <= 1.01e-8 * np.linalg.norm(b)
