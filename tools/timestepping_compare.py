#!/usr/bin/env python
"""SURVEY N4 / PAPER.md:822-834: monolithic space-time Newton-Krylov-WRMG against
sequential timestepping (Newton per timestep, FGMRES preconditioned by the same
multigrid on the one-slab problem) for the lid-driven cavity, temporal degree 0,
spatial degree 1 (P2-P1), R = 10, t in [0, 0.02], N = 20, Chebyshev V(2,2), both on
one B200 through the C ABI.  The timestepping run hands each slab's end state to
the next slab through wrmg_rhs_initial (the DG jump, R7).  Prints one JSON line.
Usage: timestepping_compare.py [Mref]"""
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
    n, N, T, R, k, q = 10 * 2 ** Mref, 20, 0.02, 10.0, 1, 0
    kw = dict(degree=k, q=q, dt=T / N, ncoarse=10, problem="ns", reynolds=R, bc="lid", weights="none", nu_pre=2,
              nu_post=2, smoother="chebyshev")
    # monolithic space-time
    torch.cuda.synchronize()
    t0 = time.time()
    c = w.Context(n, n, 1.0 / n, nslabs=N, **kw)
    U = c.zeros()
    its, lin, st = c.newton(U, rtol=1e-8, maxit=20)
    torch.cuda.synchronize()
    t_mono = time.time() - t0
    lay = c.layout
    ns_ = lay["ndof"] // (N * (q + 1))
    end_mono = U.view(ns_, N, q + 1)[:, N - 1, q].clone()
    c.close()
    # sequential timestepping: one slab per solve, end state -> next slab's initial state
    torch.cuda.synchronize()
    t0 = time.time()
    c1 = w.Context(n, n, 1.0 / n, nslabs=1, **kw)
    u0 = c1.zeros()[:ns_].clone()
    u0.zero_()
    tot_newton, tot_lin, statuses = 0, 0, set()
    for step in range(N):
        rhs = c1.zeros()
        c1.rhs_initial(u0, rhs)
        Us = c1.zeros()
        i2, l2, s2 = c1.newton(Us, rtol=1e-8, maxit=20, rhs=rhs)
        tot_newton += i2
        tot_lin += l2
        statuses.add(s2)
        u0 = Us.view(ns_, 1, q + 1)[:, 0, q].clone()
    torch.cuda.synchronize()
    t_step = time.time() - t0
    c1.close()
    diff = float(torch.linalg.norm(u0 - end_mono) / torch.linalg.norm(end_mono))
    print(json.dumps({"Mref": Mref, "mesh": n, "N": N, "R": R, "spatial": k, "temporal": q,
                      "monolithic": {"seconds": round(t_mono, 3), "newton": its, "linear": lin, "status": st},
                      "timestepping": {"seconds": round(t_step, 3), "newton_total": tot_newton,
                                       "linear_total": tot_lin, "status": sorted(statuses)},
                      "end_state_rel_diff": diff}), flush=True)


if __name__ == "__main__":
    main()
