"""The host Hessenberg eigensolver behind the Chebyshev eigenvalue estimate
(R-cheb) against LAPACK (numpy.linalg.eigvals), no device needed."""
import numpy as np
import pytest


@pytest.mark.parametrize("n,seed", [(1, 0), (2, 1), (5, 2), (20, 3), (50, 4), (50, 5)])
def test_hessenberg_eigenvalues_match_lapack(n, seed):
    import paper_2407_13997_b200 as w
    rng = np.random.default_rng(seed)
    H = np.triu(rng.standard_normal((n, n)), -1)
    if seed == 5:  # Arnoldi-like: positive subdiagonal, dominant real spectrum
        H = np.triu(rng.random((n, n)), -1) + 3 * np.eye(n)
    wr = np.zeros(n)
    wi = np.zeros(n)
    st = w.lib.wrmg_hessenberg_eig(np.ascontiguousarray(H).ctypes.data, n, wr.ctypes.data, wi.ctypes.data)
    assert st == 0
    got = np.sort_complex(wr + 1j * wi)
    ref = np.sort_complex(np.linalg.eigvals(H))
    assert np.allclose(got, ref, rtol=1e-10, atol=1e-10 * np.abs(ref).max())
    assert abs(np.abs(got).max() - np.abs(ref).max()) <= 1e-12 * np.abs(ref).max()
