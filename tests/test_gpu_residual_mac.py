"""GPU parity of the macro-block residual (kernels_residual_mac.cu), which runs on
levels with >= 5000 lattice nodes: full vectors against the oracle's explicit
space-time operator (r = b - A u, eq. heatfem, R1-R5) and y = A u, for P1 / P2 / P3
in space, DG0 ... DG3 in time (the TMA form for P1 / P2 at every q and P3 at q <= 1,
the L1 form for P3 x DG2 / DG3), slab counts that leave a ragged last 16-slab chunk,
and Neumann boundaries (boundary rows go through the fix-up kernel k_residual_rows)."""
import numpy as np
import pytest

import wrmg_inputs as wi
from test_gpu_parity import _dev, _host, assert_parity

pytestmark = pytest.mark.gpu

CASES = [  # n, k, q, N, bc
    (80, 3, 1, 7, "dirichlet0"),
    (80, 3, 0, 37, "dirichlet0"),
    (80, 3, 2, 5, "dirichlet0"),
    (80, 3, 3, 3, "dirichlet0"),
    (112, 2, 1, 9, "dirichlet0"),
    (112, 2, 1, 5, "neumann"),
    (224, 1, 0, 40, "dirichlet0"),
    (224, 1, 1, 3, "neumann"),
    (80, 3, 1, 4, "neumann"),
    # TMA form with 3 and 4 values per lane (P1 / P2 x DG2, DG3)
    (112, 2, 2, 4, "dirichlet0"),
    (112, 2, 3, 3, "neumann"),
    (224, 1, 2, 5, "dirichlet0"),
    (224, 1, 3, 3, "dirichlet0"),
    # levels between 5000 and 50 000 nodes (the macro kernel runs from 5000)
    (32, 3, 1, 9, "dirichlet0"),
    (40, 2, 2, 6, "neumann"),
]


@pytest.mark.parametrize("n,k,q,N,bc", CASES)
def test_macro_block_residual(n, k, q, N, bc):
    import paper_2407_13997_b200 as w
    from oracle import heat
    p = heat.unit_square_problem(n, k, q, N, 1.0 / N, bc="neumann" if bc == "neumann" else "dirichlet")
    assert p.nnode >= 5000  # the macro-block kernel's level-size condition
    c = w.Context(n, n, 1.0 / n, degree=k, q=q, nslabs=N, dt=1.0 / N, bc=bc)
    u = wi.spacetime_field(p.nnode, N, q, seed=11)
    b = wi.spacetime_field(p.nnode, N, q, seed=12)
    r = c.empty()
    c.residual(_dev(u), _dev(b), r)
    assert_parity(_host(r), p.residual(u, b), what="residual")
    y = c.empty()
    c.apply(_dev(u), y)
    assert_parity(_host(y), p.A @ u, what="apply")
    c.close()
