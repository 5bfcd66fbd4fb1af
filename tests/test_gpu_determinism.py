"""The two weighted-additive-scatter variants of the heat sweep (H8; SURVEY 8(a),
SPEC.md:451): FP64 atomics (default) and the coloured scatter (three passes, one
per vertex colour (i - j) mod 3; patches of one colour share no DoF, so every value
receives one addition per pass in a fixed order).  The coloured sweep is bitwise
reproducible run to run and agrees with the atomic one to rounding (1e-13), and
both agree with the oracle (the atomic path's parity is in test_gpu_parity.py)."""
import numpy as np
import pytest

import wrmg_inputs as wi
from test_gpu_parity import _dev, _host, assert_parity

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n,k,q,N", [(32, 3, 1, 40), (32, 2, 2, 9), (16, 1, 0, 16), (48, 2, 1, 20)])
def test_coloured_scatter_deterministic_and_equal_to_atomic(n, k, q, N):
    import paper_2407_13997_b200 as w
    ctx = {m: w.Context(n, n, 1.0 / n, degree=k, q=q, nslabs=N, dt=1.0 / N, scatter=m) for m in ("atomic", "colour")}
    nnode = ctx["atomic"].layout["nnode"]
    b = _dev(wi.spacetime_field(nnode, N, q, 0))
    u0 = wi.spacetime_field(nnode, N, q, 3) * 1e-2
    out = {}
    for m, c in ctx.items():
        runs = []
        for _ in range(2):
            u = _dev(u0)
            c.smooth(u, b, 2, 0.9)
            z = c.empty()
            c.vcycle(b, z)
            runs.append((_host(u), _host(z)))
        out[m] = runs
    cu, cz = out["colour"][0]
    assert np.array_equal(cu, out["colour"][1][0]) and np.array_equal(cz, out["colour"][1][1])  # bitwise
    au, az = out["atomic"][0]
    assert_parity(cu, au, tol=1e-13, what="sweeps colour vs atomic")
    assert_parity(cz, az, tol=1e-12, what="V-cycle colour vs atomic")
    for c in ctx.values():
        c.close()


def test_coloured_scatter_matches_oracle():
    """The coloured sweep against the oracle's additive sweep (R11)."""
    import paper_2407_13997_b200 as w
    from oracle import heat, patches, smoother
    n, k, q, N = 8, 3, 1, 37
    p = heat.unit_square_problem(n, k, q, N, 1.0 / N)
    c = w.Context(n, n, 1.0 / n, degree=k, q=q, nslabs=N, dt=1.0 / N, scatter="colour")
    P, _ = patches.vertex_star_patches(p.mesh, k, p.constrained)
    fac = smoother.PatchFactors(p, p.A, P)
    wts = smoother.weights(P, p.nnode)
    b = p.rhs(wi.spacetime_field(p.nnode, N, q, 0))
    u0 = wi.spacetime_field(p.nnode, N, q, 2) * ~p.con_st
    u_ref, u = u0.copy(), _dev(u0)
    for s, om in enumerate((0.7, 1.0)):
        u_ref = smoother.wr_sweep(p, p.A, u_ref, b, fac, om, wts)
        c.smooth(u, _dev(b), 1, om)
        assert_parity(_host(u), u_ref, what=f"coloured sweep {s}")
    c.close()
