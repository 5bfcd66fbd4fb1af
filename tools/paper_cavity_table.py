#!/usr/bin/env python
"""The paper's lid-driven cavity iteration table on the GPU:
Newton-FGMRES-WRMG with Chebyshev V(2,2), Vanka+star, Eisenstat-Walker forcing,
t in [0, 0.02], N = 20.  Usage: paper_cavity_table.py Mref [pressure degrees...]"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    import paper_2407_13997_b200 as w
    Mref = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    ks = [int(a) for a in sys.argv[2:]] or [1]
    printed = {}
    for line in open(os.path.join(ROOT, "tests", "golden", "paper_cavity_iterations.txt")):
        if line.strip() and not line.startswith("#"):
            m, k, q, R, nn, nl = line.split()
            printed[(int(m), int(k), int(q), float(R))] = (int(nn), int(nl))
    n, N, T = 10 * 2 ** Mref, 20, 0.02
    for k in ks:
        for q in (1, 0):
            for R in (1.0, 10.0, 100.0):
                t0 = time.time()
                c = w.Context(n, n, 1.0 / n, degree=k, q=q, nslabs=N, dt=T / N, ncoarse=10, problem="ns",
                              reynolds=R, bc="lid", weights=os.environ.get("WRMG_WEIGHTS", "none"), nu_pre=2,
                              nu_post=2, smoother="chebyshev")
                U = c.zeros()
                torch.cuda.synchronize()
                t1 = time.time()
                its, lin, st = c.newton(U, rtol=1e-8, maxit=20)
                torch.cuda.synchronize()
                t2 = time.time()
                print(json.dumps({"Mref": Mref, "pressure_degree": k, "temporal": q, "R": R,
                                  "newton": its, "linear": lin, "printed": printed.get((Mref, k, q, R)),
                                  "status": st, "ndof": c.layout["ndof"], "setup_s": round(t1 - t0, 2),
                                  "solve_s": round(t2 - t1, 2)}), flush=True)
                c.close()


if __name__ == "__main__":
    main()
