"""Finding probe (oracle only, CPU): does a multiplicative colour-by-colour Vanka+star
sweep make the C3-like V(1,1) contract where the paper's additive sweep does not
(DESIGN.md 1b finding)?  Vertex colours (i + 3 j) mod 7; within a colour the patches
are applied additively with the POU weights, colours in sequence with a fresh residual.
Prints the stationary V(1,1) residual-reduction factor per cycle for both smoothers."""
import sys

import numpy as np

sys.path.insert(0, ".")
import wrmg_inputs as wi  # noqa: E402
from oracle import ns, smoother, transfer  # noqa: E402


def mult_sweep(H, l, u, b, omega, colours):
    p, A, F, w = H.probs[l], H.A[l], H.factors[l], H.w[l]
    for col in colours:
        r = b - A @ u
        du = np.zeros_like(u)
        for pi in col:
            I_p = F.I[pi]
            x = F.solve(pi, r[I_p])
            wt = np.repeat(w[F.patches[pi]], p.q + 1)
            du[I_p] += np.tile(wt, p.N) * x
        u = p.project_pressure(u + omega * du)
    return u


def vcycle_mult(H, r, colours, l=None):
    if l is None:
        l = len(H.probs) - 1
    p = H.probs[l]
    if l == 0:
        return H.coarse(r)
    A = H.A[l]
    u = mult_sweep(H, l, np.zeros_like(r), r, H.omega_mg, colours[l])
    res = r - A @ u
    ec = vcycle_mult(H, H.probs[l - 1].project_pressure(transfer.restrict(H.P0[l], res, p.NT)), colours, l - 1)
    u = u + transfer.prolong(H.P0[l], ec, p.NT)
    return mult_sweep(H, l, u, r, H.omega_mg, colours[l][::-1])


def main(n=16, k=1, q=1, N=8, R=100.0, omega=0.8, cycles=6):
    dt = 1.0 / N
    W = wi.wind_state(n, n, 1.0 / n, k, N, q, dt)
    H = ns.NSHierarchy(n, n, 1.0 / n, k, q, N, dt, R, W=W, bc="lid", omega_mg=omega)
    colours = [None]
    for l in range(1, len(H.probs)):
        p = H.probs[l]
        _, verts = ns.vanka_star_patches(p)
        nv = p.mesh.nx + 1
        cl = [[] for _ in range(7)]
        for pi, v in enumerate(verts):
            i, j = int(v) % nv, int(v) // nv
            cl[(i + 3 * j) % 7].append(pi)
        colours.append([c for c in cl if c])
    p = H.fine
    b = p.project_pressure(np.where(p.con_st, 0.0, wi.spacetime_field(p.ns, N, q, 0)))
    for name, V in (("additive", lambda r: ns.vcycle(H, r)), ("multiplicative", lambda r: vcycle_mult(H, r, colours))):
        u = np.zeros(p.ndof)
        r0 = np.linalg.norm(b)
        hist = []
        for _ in range(cycles):
            u = u + V(b - H.A[-1] @ u)
            hist.append(np.linalg.norm(p.project_pressure(b - H.A[-1] @ u)) / r0)
        rates = [hist[0]] + [hist[i] / hist[i - 1] for i in range(1, len(hist))]
        print(f"{name:15s} n={n} R={R} omega={omega}: relres " + " ".join(f"{h:.2e}" for h in hist)
              + "  | per-cycle " + " ".join(f"{x:.2f}" for x in rates), flush=True)


if __name__ == "__main__":
    a = [float(x) for x in sys.argv[1:]]
    main(*(int(a[0]), 1, 1, int(a[1]), a[2], a[3]) if a else ())
