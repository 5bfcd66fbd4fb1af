#!/usr/bin/env python
"""C4's discretisation (BASELINE configs[3]: Newton-Krylov-WRMG, P3-P2 x DG1,
lid-driven cavity on t in [0, 1], zero initial state) at a reduced mesh that fits
the stored-inverse mode, for Re in a continuation ladder (R26).  Prints one JSON
line per run.  Usage: c4_reduced.py n N [chebyshev|damped] [--continuation] [--re 100,300]"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    import paper_2407_13997_b200 as w
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 16
    N = int(sys.argv[2]) if len(sys.argv) > 2 else 16
    sm = sys.argv[3] if len(sys.argv) > 3 and not sys.argv[3].startswith("--") else "chebyshev"
    prev = None
    res = (100.0, 300.0, 1000.0)
    if "--re" in sys.argv:
        res = tuple(float(x) for x in sys.argv[sys.argv.index("--re") + 1].split(","))
    for R in res:
        kw = dict(nu_pre=2, nu_post=2, smoother="chebyshev", weights="none") if sm == "chebyshev" else dict(
            omega_mg=0.8)
        t0 = time.time()
        c = w.Context(n, n, 1.0 / n, degree=2, q=1, nslabs=N, dt=1.0 / N, problem="ns", reynolds=R, bc="lid", **kw)
        U = c.zeros()
        if prev is not None and "--continuation" in sys.argv:  # R26: start from the previous Reynolds number
            U.copy_(prev)
        its, lin, st = c.newton(U, rtol=1e-8, maxit=15)
        prev = U.clone()
        torch.cuda.synchronize()
        print(json.dumps({"mesh": n, "N": N, "R": R, "smoother": sm, "continuation": "--continuation" in sys.argv,
                          "newton": its, "linear": lin, "status": st,
                          "ndof": c.layout["ndof"], "seconds": round(time.time() - t0, 2)}), flush=True)
        c.close()


if __name__ == "__main__":
    main()
