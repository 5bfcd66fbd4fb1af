"""Edge cases of the CUDA path against the oracle (single slab, tiny and
rectangular meshes, one-level hierarchies, zero right-hand sides, one-row
patches) and the C ABI's argument checking."""
import ctypes

import numpy as np
import pytest

import wrmg_inputs as wi

pytestmark = pytest.mark.gpu

TOL = 1e-10


def _dev(x):
    import torch
    return torch.as_tensor(np.ascontiguousarray(x), dtype=torch.float64, device="cuda:0")


def _host(t):
    import torch
    torch.cuda.synchronize()
    return t.cpu().numpy()


def _rel(a, b):
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / nb if nb > 0 else np.linalg.norm(a)


@pytest.mark.parametrize("nx,ny,k,q,N", [(8, 4, 2, 1, 1), (2, 2, 1, 0, 3), (12, 6, 1, 3, 2), (4, 8, 3, 0, 1),
                                         (6, 6, 2, 2, 33)])
def test_heat_edge_shapes(nx, ny, k, q, N):
    """Single slab (no jump), 2x2 mesh (one free node, one level), rectangular
    lattices in both orientations, a 33-slab ragged chunk: residual, two sweeps and
    a V-cycle against the oracle."""
    import paper_2407_13997_b200 as w
    from oracle import multigrid, smoother
    h = 1.0 / ny
    dt = 1.0 / N
    H = multigrid.Hierarchy(nx, ny, h, k, q, N, dt)
    p = H.fine
    c = w.Context(nx, ny, h, degree=k, q=q, nslabs=N, dt=dt)
    f = wi.spacetime_field(p.nnode, N, q, 2)
    b = c.empty()
    c.rhs(_dev(f), b)
    bref = p.rhs(f)
    assert _rel(_host(b), bref) <= TOL
    u = c.zeros()
    uref = np.zeros(p.ndof)
    L = H.levels[-1]
    for _ in range(2):
        c.smooth(u, b, 1, 1.0)
        uref = smoother.wr_sweep(p, p.A, uref, bref, L.factors, 1.0, L.w)
    assert _rel(_host(u), uref) <= TOL
    r = c.empty()
    c.residual(u, b, r)
    rref = bref - p.A @ uref
    # one free DoF (2x2 mesh): the sweep is an exact solve and r is rounding noise
    scale = max(np.linalg.norm(rref), 1e-6 * np.linalg.norm(bref))
    assert np.linalg.norm(_host(r) - rref) / scale <= TOL
    z = c.empty()
    c.vcycle(r, z)
    zref = multigrid.vcycle(H, rref)
    assert np.linalg.norm(_host(z) - zref) / max(np.linalg.norm(zref), 1e-6 * np.linalg.norm(uref)) <= TOL
    c.close()


def test_zero_rhs_gives_zero_cycle_and_zero_solution():
    """P15: b = 0 gives z = 0; FGMRES returns immediately with x = 0."""
    import paper_2407_13997_b200 as w
    c = w.Context(8, 8, 1.0 / 8, degree=2, q=1, nslabs=4, dt=0.25)
    z = c.empty()
    c.vcycle(c.zeros(), z)
    assert np.all(_host(z) == 0.0)
    x = c.empty()
    its, rel, st = c.fgmres(c.zeros(), x)
    assert st == "WRMG_OK" and its == 0 and np.all(_host(x) == 0.0)
    c.close()


def test_abi_rejects_bad_arguments():
    import paper_2407_13997_b200 as w
    c = w.Context(4, 4, 0.25, degree=1, q=0, nslabs=2, dt=0.5)
    lib = w.lib
    assert lib.wrmg_residual(c._h, None, None, None, 0) == 1          # NULL vectors
    assert lib.wrmg_smooth(c._h, None, None, 1, 1.0) == 1
    assert lib.wrmg_fgmres(c._h, None, None, 0, 1, 1e-8, 0.0, None, None) == 1  # restart < 1
    assert lib.wrmg_newton(c._h, ctypes.c_void_p(1), 1e-8, 3, None, None) == 2  # heat is linear
    assert lib.wrmg_level_size(c._h, 99, ctypes.byref(ctypes.c_int64())) == 1
    assert lib.wrmg_set_boundary_values(c._h, None) == 2  # heat: Dirichlet data is the setup's
    assert lib.wrmg_set_boundary_values(None, None) == 1
    c.close()
    with pytest.raises(w.WrmgError) as e:
        w.Context(4, 4, 0.25, degree=4, q=0, nslabs=2, dt=0.5)
    assert e.value.status == 2
    with pytest.raises(w.WrmgError) as e:
        w.Context(4, 4, 0.25, degree=1, q=0, nslabs=2, dt=-1.0)
    assert e.value.status == 1
    with pytest.raises(w.WrmgError) as e:
        w.Context(4, 4, 0.25, degree=1, q=0, nslabs=2, dt=0.5, problem="ns", reynolds=0.0)
    assert e.value.status == 1
    # NS: boundary data set, then restored with NULL
    import torch
    cn = w.Context(4, 4, 0.25, degree=1, q=0, nslabs=2, dt=0.5, problem="ns", reynolds=1.0, bc="dirichlet0")
    cn.set_boundary_values(torch.zeros(cn.layout["ndof"], dtype=torch.float64, device="cuda:0"))
    cn.set_boundary_values(None)
    cn.close()


@pytest.mark.parametrize("n,k,q,N", [(80, 3, 1, 70), (112, 2, 0, 100), (80, 3, 1, 64), (80, 3, 2, 65)])
def test_large_level_residual_ragged_chunks(n, k, q, N):
    """Residual rows on lattices large enough for the TMA-tiled kernels (>= 50000
    nodes), with N around multiples of the 32-slab chunk
    (ragged last chunk, chunk boundaries; N (q+1) odd takes the cp.async variant): sampled rows
    (corner, boundary-adjacent, interior; every slab) against the oracle's row
    formula, in residual and apply mode."""
    import torch
    import paper_2407_13997_b200 as w
    from oracle import heat
    p = heat.unit_square_problem(n, k, q, N, 1.0 / N, build_matrix=False)
    ctx = w.Context(n, n, 1.0 / n, degree=k, q=q, nslabs=N, dt=1.0 / N)
    assert p.nnode >= 50000
    u = wi.spacetime_field(p.nnode, N, q, seed=3)
    b = p.rhs(wi.spacetime_field(p.nnode, N, q, seed=4))
    dev = lambda a: torch.as_tensor(a, dtype=torch.float64, device="cuda:0")
    r, y = ctx.empty(), ctx.empty()
    ctx.residual(dev(u), dev(b), r)
    ctx.apply(dev(u), y)
    torch.cuda.synchronize()
    rg, yg = r.cpu().numpy().reshape(p.nnode, -1), y.cpu().numpy().reshape(p.nnode, -1)
    L = k * n + 1
    zero = np.zeros_like(b)
    for I, J in [(0, 0), (1, 1), (2, 1), (k, k), (L // 2, L // 2 + 1), (L - 2, L - 2), (L - 1, 5), (7, L - 2)]:
        i = J * L + I
        ref = p.residual_node(i, u, b)
        assert np.max(np.abs(rg[i] - ref)) <= 1e-10 * max(np.max(np.abs(ref)), 1e-300), (I, J)
        refy = -p.residual_node(i, u, zero)
        assert np.max(np.abs(yg[i] - refy)) <= 1e-10 * max(np.max(np.abs(refy)), 1e-300), (I, J)
    ctx.close()


def test_misaligned_vectors_rejected():
    """Device vectors must be 16-byte aligned (include/wrmg.h): a view at an odd double
    offset fails loudly with WRMG_E_INVALID instead of faulting a kernel."""
    import torch

    import paper_2407_13997_b200 as w
    from paper_2407_13997_b200._lib import WrmgError
    c = w.Context(8, 8, 1.0 / 8, degree=2, q=1, nslabs=4, dt=0.25)
    n = c.layout["ndof"]
    f = c.empty()
    c.fill_uniform(f, 0, 3)
    b = c.empty()
    c.rhs(f, b)
    bb = torch.zeros(n + 1, dtype=torch.float64, device="cuda:0")
    xb = torch.zeros(n + 1, dtype=torch.float64, device="cuda:0")
    bb[1:].copy_(b)
    for call in (lambda: c.fgmres(bb[1:], xb[1:]), lambda: c.residual(xb[1:], bb[1:], c.empty()),
                 lambda: c.smooth(xb[1:], b, 1, 1.0), lambda: c.vcycle(bb[1:], c.empty())):
        with pytest.raises(WrmgError) as ei:
            call()
        assert "INVALID" in str(ei.value)
    x = c.empty()  # the aligned call still works after the rejections
    its, rel, st = c.fgmres(b, x)
    assert st == "WRMG_OK" and its > 0
    c.close()
