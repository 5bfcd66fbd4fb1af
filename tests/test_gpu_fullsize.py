"""GPU parity at BASELINE.json's full C2 size (configs[1]: 128x128 mesh, P3 x DG1,
N = 128, dt = 1/128), in the configuration bench.py times, on outputs the oracle
can compute one by one (rows of the residual, the smoother update at sampled
nodes), plus properties of the full solve.  Tolerance R23 (1e-10 relative)."""
import numpy as np
import pytest

import wrmg_inputs as wi

pytestmark = pytest.mark.gpu

N_, K_, Q_, NT_ = 128, 3, 1, 128


@pytest.fixture(scope="module")
def c2():
    import torch

    import paper_2407_13997_b200 as w
    from oracle import heat, patches
    p = heat.unit_square_problem(N_, K_, Q_, NT_, 1.0 / NT_, build_matrix=False)
    ctx = w.Context(N_, N_, 1.0 / N_, degree=K_, q=Q_, nslabs=NT_, dt=1.0 / NT_)
    f = wi.spacetime_field(p.nnode, NT_, Q_, seed=0)
    b = p.rhs(f)
    P, verts = patches.vertex_star_patches(p.mesh, K_, p.constrained)
    dev = lambda a: torch.as_tensor(a, dtype=torch.float64, device="cuda:0")
    return dict(p=p, ctx=ctx, f=f, b=b, patches=P, dev=dev, torch=torch)


def _sample_nodes(p):
    L = K_ * N_ + 1
    pick = [(0, 0), (1, 1), (2, 1), (1, 2), (3, 3), (4, 3), (5, 4), (L // 2, L // 2), (L // 2 + 1, L // 2),
            (L - 2, L - 2), (L - 2, 1), (1, L - 2), (L - 1, 7), (200, 3)]
    return [J * L + I for I, J in pick]


def test_C2_fullsize_rhs_and_residual_rows(c2):
    p, ctx, dev, torch = c2["p"], c2["ctx"], c2["dev"], c2["torch"]
    b = ctx.empty()
    ctx.rhs(dev(c2["f"]), b)
    u = wi.spacetime_field(p.nnode, NT_, Q_, seed=1)
    r = ctx.empty()
    ctx.residual(dev(u), b, r)
    torch.cuda.synchronize()
    bg, rg = b.cpu().numpy(), r.cpu().numpy()
    scale_b = np.max(np.abs(c2["b"]))
    assert np.max(np.abs(bg - c2["b"])) <= 1e-10 * scale_b  # b everywhere (oracle rhs is cheap)
    worst = 0.0
    for i in _sample_nodes(p):
        ref = p.residual_node(i, u, c2["b"])
        got = rg.reshape(p.nnode, -1)[i]
        worst = max(worst, np.max(np.abs(got - ref)) / max(np.max(np.abs(ref)), 1e-300))
    assert worst <= 1e-10, worst


def test_C2_fullsize_sweep_sampled_nodes(c2):
    """One additive sweep (omega = 1) from a random state: the update at sampled
    nodes equals omega * sum_{p ni i} x_p[i] / mu_i with x_p the oracle's exact
    patch space-time solve (Kronecker-built blocks, per-slab LAPACK LU)."""
    from oracle import patches as pm
    from oracle import smoother
    p, ctx, dev, torch = c2["p"], c2["ctx"], c2["dev"], c2["torch"]
    u0 = wi.spacetime_field(p.nnode, NT_, Q_, seed=2) * np.repeat(p.free, p.NT)
    ug = dev(u0)
    ctx.smooth(ug, dev(c2["b"]), 1, 1.0)
    torch.cuda.synchronize()
    du_gpu = (ug.cpu().numpy() - u0).reshape(p.nnode, -1)
    mu = pm.multiplicity(c2["patches"], p.nnode)
    nodes = [i for i in _sample_nodes(p) if p.free[i]]
    rcache = {}

    def rnode(j):
        if j not in rcache:
            rcache[j] = p.residual_node(j, u0, c2["b"]).reshape(NT_, Q_ + 1)
        return rcache[j]

    worst = 0.0
    for i in nodes:
        acc = np.zeros(p.NT)
        for pt in c2["patches"]:
            if i not in pt:
                continue
            g = np.concatenate([np.stack([rnode(j)[n] for j in pt]).ravel() for n in range(NT_)])
            x = smoother.patch_solve_kron(p, pt, g).reshape(NT_, pt.size, Q_ + 1)
            acc += x[:, list(pt).index(i), :].ravel() / mu[i]
        worst = max(worst, np.max(np.abs(du_gpu[i] - acc)) / np.max(np.abs(acc)))
    assert worst <= 1e-10, worst


@pytest.mark.parametrize("mode", ["auto", "lu"])
def test_C2_fullsize_solve(c2, mode):
    """FGMRES(30) + V(1,1) to 1e-8 at full size: converges, true residual below the
    tolerance, both factor modes give the same iterate and iteration count."""
    import paper_2407_13997_b200 as w
    torch = c2["torch"]
    ctx = c2["ctx"] if mode == "auto" else w.Context(N_, N_, 1.0 / N_, degree=K_, q=Q_, nslabs=NT_, dt=1.0 / NT_,
                                                     factor_mode="lu")
    b = c2["dev"](c2["b"])
    x = ctx.empty()
    its, rel, st = ctx.fgmres(b, x, restart=30, maxit=100, rtol=1e-8)
    assert st == "WRMG_OK" and rel <= 1e-8 * 1.001 and its <= 12
    r = ctx.empty()
    ctx.residual(x, b, r)
    assert float(torch.linalg.norm(r)) <= 1e-8 * 1.001 * float(torch.linalg.norm(b))
    c2.setdefault("solves", {})[mode] = (its, x.cpu().numpy())
    if len(c2["solves"]) == 2:
        (i1, x1), (i2, x2) = c2["solves"].values()
        assert i1 == i2
        assert np.linalg.norm(x1 - x2) <= 1e-9 * np.linalg.norm(x1)
