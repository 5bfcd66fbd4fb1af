"""Oracle pins P4, P5, P6, P13, P19 for the space-time heat operator
(eq. heatfem; eq. dgintime)."""
import numpy as np
import pytest
import scipy.linalg as sla
import scipy.sparse.linalg as spla

import wrmg_inputs as wi
from oracle import heat, mesh


def test_P4_dg0_is_backward_euler():
    """q = 0: the all-at-once solve equals a backward-Euler march
    (M + dt kappa K) U_n = M U_{n-1} + dt M f_n (free rows; Dirichlet 0)."""
    n, N, dt, kappa = 5, 6, 0.07, 1.3
    p = heat.unit_square_problem(n, 2, 0, N, dt, kappa=kappa)
    f = wi.spacetime_field(p.nnode, N, 0, seed=3)
    U = spla.spsolve(p.A.tocsc(), p.rhs(f)).reshape(p.nnode, N)
    fr = p.free
    Mff = p.M[fr][:, fr].toarray()
    Kff = p.K[fr][:, fr].toarray()
    Mf = p.M[fr].toarray()
    prev = np.zeros(fr.sum())
    f2 = f.reshape(p.nnode, N)
    for s in range(N):
        cur = np.linalg.solve(Mff + dt * kappa * Kff, Mff @ prev + dt * (Mf @ f2[:, s]))
        assert np.allclose(U[fr, s], cur, rtol=1e-11, atol=1e-13)
        prev = cur
    assert np.all(U[~fr] == 0.0)


PADE = {
    0: lambda z: 1.0 / (1.0 - z),
    1: lambda z: (1.0 + z / 3.0) / (1.0 - 2.0 * z / 3.0 + z * z / 6.0),
    2: lambda z: (1.0 + 2 * z / 5 + z * z / 20) / (1.0 - 3 * z / 5 + 3 * z * z / 20 - z ** 3 / 60),
}


@pytest.mark.parametrize("q", [0, 1, 2])
def test_P5_amplification_factor(q):
    """For K v = lambda M v (free block), u0 = v and no forcing, the end-of-slab
    value after n+1 slabs is R(z)^(n+1) v with R the (q, q+1) subdiagonal Pade
    approximant (Radau IIA stability function), z = -kappa lambda dt."""
    n, N, dt, kappa = 4, 5, 0.05, 0.8
    p = heat.unit_square_problem(n, 1, q, N, dt, kappa=kappa)
    fr = p.free
    lam, vecs = sla.eigh(p.K[fr][:, fr].toarray(), p.M[fr][:, fr].toarray())
    for j in (0, len(lam) // 2, len(lam) - 1):
        v = np.zeros(p.nnode)
        v[fr] = vecs[:, j]
        b = p.rhs(np.zeros(p.ndof), u0=v)
        U = spla.spsolve(p.A.tocsc(), b).reshape(p.nnode, N, q + 1)
        R = PADE[q](-kappa * lam[j] * dt)
        for s in range(N):
            end = U[:, s, q]  # phi_q(1) = 1 (q >= 1); DG0: the constant
            assert np.allclose(end, R ** (s + 1) * v, rtol=1e-9, atol=1e-12)


def test_P6_block_structure():
    q, N = 1, 4
    p = heat.unit_square_problem(3, 2, q, N, 0.1)
    A = p.A.tocoo()
    nq = q + 1
    rs = (A.row % p.NT) // nq
    cs = (A.col % p.NT) // nq
    assert np.all(cs <= rs) and np.all(rs - cs <= 1)
    # (n, n-1) block on free rows is -E1 (x) M: only a=0 rows, b=q columns
    sub = rs - cs == 1
    ra, ca = A.row[sub] % nq, A.col[sub] % nq
    assert np.all(ra == 0) and np.all(ca == q)
    i, j = A.row[sub] // p.NT, A.col[sub] // p.NT
    Md = p.M.toarray()
    assert np.allclose(A.data[sub], -Md[i, j])


def test_P19_neumann_constant_solution():
    """Natural BCs, u0 = 1, f = 0: the discrete solution is U = 1 exactly
    (constants are in the kernel of K and the jump is consistent)."""
    for q in (0, 1, 2):
        p = heat.unit_square_problem(3, 2, q, 4, 0.2, bc="neumann")
        b = p.rhs(np.zeros(p.ndof), u0=np.ones(p.nnode))
        U = spla.spsolve(p.A.tocsc(), b)
        assert np.max(np.abs(U - 1.0)) < 1e-12


def _manufactured_error(n, k, q, N, T):
    """u = sin(pi x) sin(pi y) exp(-t), f = u_t - Delta u = (2 pi^2 - 1) u;
    returns the mass-norm error of the end-of-horizon nodal values."""
    p = heat.unit_square_problem(n, k, q, N, T / N)
    xy = mesh.node_coords(p.mesh, k)
    s = np.sin(np.pi * xy[:, 0]) * np.sin(np.pi * xy[:, 1])
    tn = p.tm.nodes if q > 0 else np.array([0.5])
    times = (np.arange(N)[:, None] + tn[None, :]) * p.dt  # (N, q+1) nodal times
    if q == 0:
        # DG0: interpolate f as the slab-midpoint constant
        pass
    f = (2 * np.pi ** 2 - 1) * s[:, None, None] * np.exp(-times)[None, :, :]
    b = p.rhs(f.reshape(-1), u0=s)
    U = spla.spsolve(p.A.tocsc(), b).reshape(p.nnode, N, q + 1)
    e = U[:, -1, q] - s * np.exp(-T)
    return np.sqrt(e @ (p.M @ e))


@pytest.mark.parametrize("k", [1, 2])
def test_P13_manufactured_spatial_order(k):
    """Spatial order >= k+1 (L2) with q = 2 and small dt (temporal error
    O(dt^5) at slab ends is negligible)."""
    e1 = _manufactured_error(4, k, 2, 8, 0.1)
    e2 = _manufactured_error(8, k, 2, 8, 0.1)
    order = np.log2(e1 / e2)
    assert order >= k + 1 - 0.2, order


def test_residual_node_and_rows_match_explicit_A():
    """The row-wise evaluators used for full-size sampled parity equal b - A u."""
    p = heat.unit_square_problem(4, 3, 1, 5, 0.2)
    u = wi.spacetime_field(p.nnode, 5, 1, seed=4)
    b = wi.spacetime_field(p.nnode, 5, 1, seed=5)
    r = p.residual(u, b).reshape(p.nnode, -1)
    for i in (0, 7, 20, p.nnode // 2, p.nnode - 1):
        assert np.allclose(p.residual_node(i, u, b), r[i], rtol=1e-13, atol=1e-14)
    rows = np.array([3, 50, 77, p.ndof - 1])
    assert np.allclose(p.residual_rows(rows, u, b), r.ravel()[rows], rtol=1e-13, atol=1e-14)
