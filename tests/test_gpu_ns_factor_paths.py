"""Every Vanka block-inversion launch path against the oracle: the register-tiled kernel
(k_ns_factor_rt) at m = 39 (P2-P1 x DG0, 5 tile columns), 78 (P2-P1 x DG1, C3) and 81
(P3-P2 x DG0, 11 tile columns), and the shared-memory kernel with column-strip updates at
m = 117 (P2-P1 x DG2: odd m, scalar C accesses) and 162 (P3-P2 x DG1, C4: 16-byte C
accesses).  Three damped sweeps from u = 0 with the inverses of a wind linearisation
(R18), GPU = oracle to R23's 1e-10."""
import numpy as np
import pytest

from test_gpu_ns import _host, _rhs, _setup, assert_parity

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("k,q,N", [(1, 0, 4), (1, 1, 3), (2, 0, 3), (1, 2, 2), (2, 1, 2)])
def test_factor_paths_sweeps_match_oracle(k, q, N):
    from oracle import smoother
    c, H, W = _setup(8, k, q, N)
    p = H.fine
    b, bref = _rhs(c, p, seed=11)
    u = c.zeros()
    uref = np.zeros(p.ndof)
    for it in range(3):
        c.smooth(u, b, 1, 0.8)
        uref = p.project_pressure(smoother.wr_sweep(p, H.A[-1], uref, bref, H.factors[-1], 0.8, H.w[-1]))
        assert_parity(_host(u), uref, what=f"k={k} q={q} sweep {it}")
    c.close()
