"""Pins of the Chebyshev-accelerated V(2,2) and of the paper's
heat protocol against its printed FGMRES iteration counts (PAPER.md:533-539,
tests/golden/paper_heat_iterations.txt).  The paper reports Mref = 3, 4 (80^2,
160^2 cells); the oracle runs the same protocol on the Mref = 2 hierarchy (40^2
cells, coarsest 10^2) to stay within the CPU suite's budget (at Mref = 1 the
absolute tolerance 1e-6 sits between iterations 3 and 4 -- |g_3| = 1.5e-6 for
P1 x DG1 -- so the count there is not the printed one), and the GPU reproduces
the printed Mref = 3 table (tests/test_gpu_paper_heat.py)."""
import numpy as np
import pytest

import wrmg_inputs as wi
from oracle import krylov, multigrid, smoother
from wrmg_testutil import read_golden


def paper_problem(Mref, k, q, steps=50):
    n, N, T = 10 * 2 ** Mref, 20, 0.02
    H = multigrid.Hierarchy(n, n, 1.0 / n, k, q, N, T / N, n_coarse=10, weight_mode="none", bc="neumann",
                            nu_pre=2, nu_post=2, smoother_kind="chebyshev", cheb_steps=steps)
    p = H.fine
    b = p.rhs(np.zeros(p.ndof), u0=wi.paper_heat_u0(n, n, 1.0 / n, k))
    return H, p, b


def solve(H, p, b):
    return krylov.fgmres(lambda v: p.A @ v, lambda r: multigrid.vcycle(H, r), b, restart=30, maxit=50, rtol=1e-6,
                         atol=1e-6)


@pytest.mark.parametrize("k,q", [(1, 0), (1, 1)])
def test_paper_heat_iteration_count(k, q):
    printed = {(int(r[1]), int(r[2])): int(r[3]) for r in read_golden("paper_heat_iterations.txt")}
    H, p, b = paper_problem(2, k, q)
    x, its, hist, st = solve(H, p, b)
    assert st == "converged"
    assert its == printed[(k, q)]


def test_chebyshev_degree_one_is_optimally_damped_relaxation():
    """nu = 1: x_1 = x_0 + B r_0 / theta, theta = (0.25 + 1.05) lam / 2 -- a single
    damped sweep with omega = 1 / theta (exact identity of the recurrence)."""
    H, p, b = paper_problem(1, 1, 1, steps=10)
    L, lam = H.levels[-1], H.lam[-1]
    u0 = wi.spacetime_field(p.nnode, p.N, p.q, 3) * 1e-3
    x1 = multigrid.chebyshev(L, u0, b, lam, 1)
    ref = smoother.wr_sweep(p, p.A, u0, b, L.factors, 1.0 / (0.65 * lam), L.w)
    assert np.allclose(x1, ref, rtol=1e-13, atol=1e-18)


def test_lambda_estimate_bounds_the_relaxed_operator():
    """The Arnoldi estimate is a Ritz value of B A: of the size of the power-
    iteration growth rate of B A (which converges to the spectral radius)."""
    H, p, b = paper_problem(1, 1, 1, steps=20)
    L, lam = H.levels[-1], H.lam[-1]
    rng = np.random.default_rng(0)
    v = rng.standard_normal(p.ndof)
    for _ in range(30):
        v = multigrid.relaxation(L, p.A @ v)
        v /= np.linalg.norm(v)
    growth = np.linalg.norm(multigrid.relaxation(L, p.A @ v))
    assert 0.5 * growth <= lam <= 3.0 * growth
