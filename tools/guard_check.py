"""Out-of-bounds check without compute-sanitizer (closed on this GPU pool): run with
WRMG_GUARD=1 so every device allocation of the library carries 4 KB guard bands of
0xFF (NaN doubles, -1 indices).  Each workload below is compared with the oracle --
an out-of-bounds read of a guard poisons it -- and the bands are checked for
out-of-bounds writes when the contexts free their memory.  Prints one line per case
and the violation count; exit code 1 on any failure."""
import os
import sys
import threading

import numpy as np
import torch

sys.path.insert(0, ".")
assert os.environ.get("WRMG_GUARD") == "1", "run with WRMG_GUARD=1"
import paper_2407_13997_b200 as w  # noqa: E402
import wrmg_inputs as wi  # noqa: E402
from oracle import heat, multigrid, ns  # noqa: E402

fail = []


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def dev(a):
    return torch.as_tensor(np.ascontiguousarray(a), dtype=torch.float64, device="cuda:0")


def host(t):
    torch.cuda.synchronize()
    return t.cpu().numpy()


def heat_case(n, k, q, N, **kw):
    H = multigrid.Hierarchy(n, n, 1.0 / n, k, q, N, 1.0 / N)
    p = H.fine
    c = w.Context(n, n, 1.0 / n, degree=k, q=q, nslabs=N, dt=1.0 / N, **kw)
    b = p.rhs(wi.spacetime_field(p.nnode, N, q, 0))
    u0 = wi.spacetime_field(p.nnode, N, q, 3) * ~p.con_st
    r = c.empty()
    c.residual(dev(u0), dev(b), r)
    e1 = rel(host(r), p.residual(u0, b))
    z = c.empty()
    c.vcycle(dev(b), z)
    e2 = rel(host(z), multigrid.vcycle(H, b))
    c.close()
    print(f"heat n={n} k={k} q={q} N={N} {kw}: residual {e1:.1e} vcycle {e2:.1e}", flush=True)
    if not (e1 <= 1e-10 and e2 <= 1e-10):
        fail.append(("heat", n, k, q))


heat_case(16, 1, 0, 16)
heat_case(8, 3, 1, 37)
heat_case(32, 2, 1, 20)          # >= 1000 patches: symmetric + DMMA sweeps
heat_case(32, 2, 1, 20, scatter="colour")
heat_case(48, 3, 1, 6)           # macro-block residual (>= 5000 nodes)
heat_case(32, 2, 2, 5)

# Navier-Stokes (Taylor-Hood P2-P1 x DG1, 8x8, 3 slabs): J x and one V(1,1) at the C3 wind
n, k, q, N, R = 8, 1, 1, 3, 100.0
W = wi.wind_state(n, n, 1.0 / n, k, N, q, 1.0 / N)
c = w.Context(n, n, 1.0 / n, degree=k, q=q, nslabs=N, dt=1.0 / N, problem="ns", reynolds=R, bc="lid", omega_mg=0.8)
c.linearize(dev(W))
Hn = ns.NSHierarchy(n, n, 1.0 / n, k, q, N, 1.0 / N, R, W=W, bc="lid", omega_mg=0.8)
pn = Hn.fine
x = wi.spacetime_field(pn.ns, N, q, 7)
y = c.empty()
c.apply(dev(x), y)
e1 = rel(host(y), Hn.A[-1] @ x)
bb = x.copy()
bb[pn.con_st] = 0.0
bb = pn.project_pressure(bb)
z = c.empty()
c.vcycle(dev(bb), z)
e2 = rel(host(z), ns.vcycle(Hn, bb))
c.close()
print(f"ns: apply {e1:.1e} vcycle {e2:.1e}", flush=True)
if not (e1 <= 1e-10 and e2 <= 1e-10):
    fail.append("ns")

# strips (loopback, 4 ranks, agglomerated coarse levels): FGMRES count of one rank
P, snx, ny, k, q, N, nc = 4, 4, 16, 2, 1, 6, 2
gnx = P * snx
g = w.Context(gnx, ny, 1.0 / ny, degree=k, q=q, nslabs=N, dt=1.0 / N, ncoarse=nc)
gl = g.layout
f = wi.spacetime_field(gl["nnode"], N, q, 9)
bg = g.empty()
g.rhs(dev(f), bg)
xg = g.empty()
its_g = g.fgmres(bg, xg, restart=30, maxit=60, rtol=1e-10)[0]
g.close()
hub = w.LoopbackHub(P)
its = [None] * P


def rank_fn(r):
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        cc = w.Context(gnx, ny, 1.0 / ny, degree=k, q=q, nslabs=N, dt=1.0 / N, ncoarse=nc, rank=r, nranks=P, hub=hub,
                       stream=st.cuda_stream)
        lay = cc.layout
        fl = f.reshape(gl["ly"], gl["lx"], gl["nt"])[:, lay["g0"]:lay["g0"] + lay["lx"], :].copy()
        b = cc.empty()
        cc.rhs(torch.as_tensor(fl.reshape(-1), device="cuda:0"), b)
        xx = cc.empty()
        its[r] = cc.fgmres(b, xx, restart=30, maxit=60, rtol=1e-10)[0]
        st.synchronize()
        cc.close()


th = [threading.Thread(target=rank_fn, args=(r,)) for r in range(P)]
for t in th:
    t.start()
for t in th:
    t.join()
hub.close()
print(f"strips: fgmres its {its} vs one rank {its_g}", flush=True)
if any(i != its_g for i in its):
    fail.append("strips")

v = w.guard_violations()
print(f"guard violations {v}; failures {fail}")
sys.exit(1 if (v or fail) else 0)
