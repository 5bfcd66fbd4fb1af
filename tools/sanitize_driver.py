"""Small driver for compute-sanitizer runs (memcheck / racecheck / synccheck) over
every kernel family of the hot path: C1 (P1 x DG0, 16^2, N = 16: class-stencil
residual, chunk-parallel Kronecker sweep, coarse solve, FGMRES), a P3 x DG1 level
above the macro-kernel and symmetric-sweep thresholds (80^2, N = 8: TMA macro
residual, symmetric sweep, DMMA Kronecker sweep for the boundary classes, coloured
scatter), a 16^2 C3-shaped Navier-Stokes problem (P2-P1 x DG1, N = 4, Re 100:
assembly, block inversion, Vanka sweep, pinned coarse solve, Newton-Krylov) and a
two-rank loopback strip run with agglomerated coarse levels."""
import sys
import threading

import torch

sys.path.insert(0, ".")
import paper_2407_13997_b200 as w  # noqa: E402
import wrmg_inputs as wi  # noqa: E402


def heat(n, k, q, N, **kw):
    c = w.Context(n, n, 1.0 / n, degree=k, q=q, nslabs=N, dt=1.0 / N, **kw)
    f = c.empty()
    c.fill_uniform(f, 0, 0)
    b = c.empty()
    c.rhs(f, b)
    u = c.zeros()
    c.smooth(u, b, 2, 1.0)
    r = c.empty()
    c.residual(u, b, r)
    z = c.empty()
    c.vcycle(r, z)
    x = c.empty()
    its, rel, st = c.fgmres(b, x, restart=30, maxit=4, rtol=1e-8)
    torch.cuda.synchronize()
    c.close()
    return its


print("C1", heat(16, 1, 0, 16))
print("P3xDG1 80^2", heat(80, 3, 1, 8))
print("P3xDG1 80^2 coloured", heat(80, 3, 1, 8, scatter="colour"))
print("P2xDG2 48^2", heat(48, 2, 2, 5))

n, k, q, N = 16, 1, 1, 4
c = w.Context(n, n, 1.0 / n, degree=k, q=q, nslabs=N, dt=1.0 / N, problem="ns", reynolds=100.0, bc="lid",
              omega_mg=0.8)
W = torch.as_tensor(wi.wind_state(n, n, 1.0 / n, k, N, q, 1.0 / N), device="cuda:0")
c.linearize(W)
f = c.empty()
c.fill_uniform(f, 0, 0)
b = c.empty()
c.rhs(f, b)
u = c.zeros()
c.smooth(u, b, 2, 1.0)
z = c.empty()
c.vcycle(b, z)
U = c.zeros()
print("NS newton", c.newton(U, rtol=1e-6, maxit=2))
torch.cuda.synchronize()
c.close()

P, gnx, ny = 2, 8, 8
hub = w.LoopbackHub(P)


def rank(r):
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        cc = w.Context(gnx, ny, 1.0 / ny, degree=2, q=1, nslabs=6, dt=1.0 / 6, ncoarse=2, rank=r, nranks=P, hub=hub,
                       stream=st.cuda_stream)
        ff = cc.empty()
        cc.fill_uniform(ff, 0, 0)
        bb = cc.empty()
        cc.rhs(ff, bb)
        xx = cc.empty()
        cc.fgmres(bb, xx, restart=30, maxit=5, rtol=1e-8)
        st.synchronize()
        cc.close()


th = [threading.Thread(target=rank, args=(r,)) for r in range(P)]
for t in th:
    t.start()
for t in th:
    t.join()
hub.close()
print("ok")
