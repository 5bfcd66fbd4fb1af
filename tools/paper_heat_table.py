#!/usr/bin/env python
"""The paper's heat iteration table on the GPU: every
(spatial 1..3, temporal 0..3) pair at Mref = 3 (and optionally 4), Chebyshev
V(2,2), FGMRES rtol/atol 1e-6.  Prints one JSON line per case and a summary
against tests/golden/paper_heat_iterations.txt."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    import paper_2407_13997_b200 as w
    import wrmg_inputs as wi
    mrefs = [int(a) for a in sys.argv[1:]] or [3]
    printed = {}
    for line in open(os.path.join(ROOT, "tests", "golden", "paper_heat_iterations.txt")):
        if line.strip() and not line.startswith("#"):
            m, k, q, its = (int(x) for x in line.split())
            printed[(m, k, q)] = its
    for Mref in mrefs:
        for k in (1, 2, 3):
            for q in (0, 1, 2, 3):
                n, N, T = 10 * 2 ** Mref, 20, 0.02
                t0 = time.time()
                c = w.Context(n, n, 1.0 / n, degree=k, q=q, nslabs=N, dt=T / N, ncoarse=10, weights="none",
                              bc="neumann", nu_pre=2, nu_post=2, smoother="chebyshev", cheb_steps=50)
                torch.cuda.synchronize()
                t1 = time.time()
                b = c.zeros()
                c.rhs_initial(torch.as_tensor(wi.paper_heat_u0(n, n, 1.0 / n, k), device="cuda:0"), b)
                x = c.empty()
                torch.cuda.synchronize()
                t2 = time.time()
                its, rel, st = c.fgmres(b, x, restart=30, maxit=50, rtol=1e-6, atol=1e-6)
                torch.cuda.synchronize()
                t3 = time.time()
                lam = [round(c.cheb_lambda(l), 4) for l in range(1, c.layout["nlevels"])]
                print(json.dumps({"Mref": Mref, "spatial": k, "temporal": q, "dofs": c.layout["ndof"],
                                  "iterations": its, "printed": printed.get((Mref, k, q)), "status": st,
                                  "relres": rel, "lambda": lam, "setup_s": round(t1 - t0, 2),
                                  "solve_s": round(t3 - t2, 4)}), flush=True)
                c.close()


if __name__ == "__main__":
    main()
