"""Pin P11: the oracle's spaces and sparsity against the paper's printed DoF and
nonzero counts (tables tab:heat:dof_nnz3 / dof_nnz4),
and the shared input generator against the published splitmix64 sequence.

DoFs = (k n + 1)^2 N (q + 1) for CG(k) x DG(q) on the n x n mesh (n = 10 * 2^Mref,
PAPER.md:524-526; N = 20).  The paper's nonzero counts are
reproduced by the pattern "coupled across 3 timesteps":
nnz = nnz_s (q + 1)^2 (3N - 2), nnz_s the spatial finite-element sparsity
(pairs of nodes sharing a cell).  DESIGN.md reading R-census.
"""
import numpy as np
import pytest

import wrmg_inputs as wi
from oracle import fem, mesh
from wrmg_testutil import read_golden

# Printed 5.9e7 differs from every consistent count (5.69e7); the Mref=4 entry of
# the same column agrees.  Treated as a typo in the paper (DESIGN.md R-census).
KNOWN_TYPO = {(3, 0, 3)}


def _spatial_pattern_nnz(n, k):
    m = mesh.unit_square(n)
    d = fem.cell_dofs(m, k)
    L = (k * n + 1) ** 2
    r = np.repeat(d, d.shape[1], axis=1).ravel()
    c = np.tile(d, (1, d.shape[1])).ravel()
    return np.unique(r * L + c).size, L


def _two_sf(x):
    return float(f"{x:.1e}")


@pytest.mark.parametrize("mref", [3, 4])
def test_P11_heat_census(mref):
    N = 20
    rows = [r for r in read_golden("census_heat.txt") if int(r[0]) == mref]
    assert rows
    cache = {}
    for _, q, k, dofs, nnz in rows:
        q, k = int(q), int(k)
        n = 10 * 2 ** mref
        if k not in cache:
            cache[k] = _spatial_pattern_nnz(n, k)
        nnz_s, L = cache[k]
        my_dofs = L * N * (q + 1)
        my_nnz = nnz_s * (q + 1) ** 2 * (3 * N - 2)
        assert _two_sf(my_dofs) == float(dofs), (mref, q, k)
        if (mref, q, k) in KNOWN_TYPO:
            assert _two_sf(my_nnz) != float(nnz)
            continue
        assert _two_sf(my_nnz) == float(nnz), (mref, q, k, my_nnz)


def test_P11_spatial_nnz_exact():
    # 80 x 80 mesh spatial pattern sizes (DESIGN.md census reading)
    assert _spatial_pattern_nnz(80, 1)[0] == 45281
    assert _spatial_pattern_nnz(80, 2)[0] == 295681


def test_inputs_splitmix64_reference_values():
    """splitmix64 seeded at 0: outputs 0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4
    (the published reference sequence); id g, seed s uses state g + (s+1) G."""
    v = wi.uniform_pm1([0], seed=0)[0]
    assert v == 2.0 * (0xE220A8397B1DCDAF >> 11) * 2.0 ** -53 - 1.0
    v = wi.uniform_pm1([0], seed=1)[0]
    assert v == 2.0 * (0x6E789E6AA1B965F4 >> 11) * 2.0 ** -53 - 1.0
    x = wi.uniform_pm1(np.arange(100000, dtype=np.uint64))
    assert x.min() >= -1.0 and x.max() < 1.0 and abs(x.mean()) < 0.01
