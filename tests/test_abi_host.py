"""CPU tests of the C-ABI library: it loads without a GPU, exports every entry
point include/wrmg.h declares, and its host-side setup logic (H3 patch tables,
level sizes) agrees with the oracle.  No compute call touches a device here."""
import ctypes
import os
import re

import numpy as np
import pytest

from oracle import heat, mesh, multigrid, patches

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _header_functions():
    src = open(os.path.join(ROOT, "include", "wrmg.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(wrmg_[a-z_]+)\s*\(", src)))


def test_library_loads_and_exports_header_symbols():
    import paper_2407_13997_b200 as w
    names = _header_functions()
    assert len(names) >= 15
    for n in names:
        assert hasattr(w.lib, n), n  # ctypes resolves the symbol in libwrmg.so
    assert set(names) == set(w.exported_symbols())


def test_errors_without_device_are_reported():
    import paper_2407_13997_b200 as w
    with pytest.raises(w.WrmgError) as e:
        w.wrmg_plan(4, 4, 0.25, 5, 0, 4)  # unsupported degree
    assert e.value.status == 2


@pytest.mark.parametrize("n,k", [(4, 1), (5, 2), (4, 3), (6, 3)])
def test_patch_tables_match_oracle(n, k):
    import paper_2407_13997_b200 as w
    nodes, sizes = w.wrmg_plan_patches(n, n, 1.0 / n, k)
    p = heat.unit_square_problem(n, k, 0, 1, 1.0, build_matrix=False)
    P, _ = patches.vertex_star_patches(p.mesh, k, p.constrained)
    assert len(P) == nodes.shape[0]
    for pt, row, s in zip(P, nodes, sizes):
        assert s == pt.size
        assert np.array_equal(row[:s], pt)
        assert np.all(row[s:] == -1)


@pytest.mark.parametrize("n,k,q,N", [(16, 1, 0, 16), (128, 3, 1, 128), (1024, 2, 1, 256), (12, 2, 2, 5)])
def test_plan_sizes(n, k, q, N):
    import paper_2407_13997_b200 as w
    lay = w.wrmg_plan(n, n, 1.0 / n, k, q, N)
    assert lay["nnode"] == (k * n + 1) ** 2
    assert lay["nfree_st"] == (k * n - 1) ** 2 * N * (q + 1)
    assert lay["ndof"] == lay["nnode"] * N * (q + 1)
    assert lay["mp_max"] == {1: 1, 2: 7, 3: 19}[k]
    nl = 1
    m = n
    while m > 4 and m % 2 == 0:
        m //= 2
        nl += 1
    assert lay["nlevels"] == nl
