"""Right-preconditioned flexible GMRES.

"We use standard geometric multigrid V-cycles as preconditioners for FGMRES,
where we use FGMRES ... because it explicitly stores the preconditioned Arnoldi
vectors and, thus, can reassemble the final solution without the additional
application of the preconditioner."  DESIGN.md R16: x0 = 0, restart 30, classical
Gram-Schmidt (one pass, orth="cgs": the default orthogonalisation of the PETSc
FGMRES behind the paper's Firedrake runs; orth="cgs2" applies it
twice), Givens rotations, stop when the implicit residual |g_{j+1}| <= max(rtol
||b||, atol); true residual recomputed at each restart; breakdown when h_{j+1,j} <
1e-30 (reported separately).
Textbook algorithm (Saad, FGMRES), written out step by step.
"""
import numpy as np


def fgmres(A, M, b, restart=30, maxit=200, rtol=1e-8, atol=0.0, x0=None, orth="cgs"):
    """Returns (x, iterations, history, status) with status in
    {'converged', 'breakdown', 'maxit'}; history holds |g_{j+1}| per iteration
    (history[0] = initial residual norm)."""
    b = np.asarray(b, dtype=float)
    x = np.zeros_like(b) if x0 is None else np.array(x0, dtype=float)
    bnorm = np.linalg.norm(b)
    target = max(rtol * bnorm, atol)
    r = b - A(x) if x0 is not None else b.copy()
    beta = np.linalg.norm(r)
    hist = [beta]
    if beta <= target:
        return x, 0, hist, "converged"
    its = 0
    status = "maxit"
    while its < maxit:
        V = [r / beta]
        Z = []
        H = np.zeros((restart + 1, restart))
        cs, sn = np.zeros(restart), np.zeros(restart)
        g = np.zeros(restart + 1)
        g[0] = beta
        j_end = 0
        done = False
        for j in range(restart):
            Z.append(M(V[j]))
            w = A(Z[j])
            Vm = np.array(V)  # (j+1, n)
            h = Vm @ w
            w = w - Vm.T @ h
            if orth == "cgs2":
                h2 = Vm @ w
                w = w - Vm.T @ h2
                h = h + h2
            elif orth != "cgs":
                raise ValueError(orth)
            hn = np.linalg.norm(w)
            col = np.zeros(restart + 1)
            col[:j + 1] = h
            col[j + 1] = hn
            for i in range(j):
                t = cs[i] * col[i] + sn[i] * col[i + 1]
                col[i + 1] = -sn[i] * col[i] + cs[i] * col[i + 1]
                col[i] = t
            d = np.hypot(col[j], col[j + 1])
            cs[j], sn[j] = col[j] / d, col[j + 1] / d
            col[j] = d
            col[j + 1] = 0.0
            g[j + 1] = -sn[j] * g[j]
            g[j] = cs[j] * g[j]
            H[:, j] = col
            its += 1
            j_end = j + 1
            hist.append(abs(g[j + 1]))
            if hn < 1e-30:
                status, done = "breakdown", True
                break
            V.append(w / hn)
            if abs(g[j + 1]) <= target:
                status, done = "converged", True
                break
            if its >= maxit:
                done = True
                break
        y = np.zeros(j_end)
        for i in range(j_end - 1, -1, -1):
            y[i] = (g[i] - H[i, i + 1:j_end] @ y[i + 1:]) / H[i, i]
        for i in range(j_end):
            x = x + y[i] * Z[i]
        if done:
            return x, its, hist, status
        r = b - A(x)
        beta = np.linalg.norm(r)
        if beta <= target:
            return x, its, hist, "converged"
    return x, its, hist, status
