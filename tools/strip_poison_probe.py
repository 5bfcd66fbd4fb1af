"""Probe for reads of uninitialised user-vector memory on the strip path: the loopback FGMRES
of tools/guard_check.py with b's unwritten entries and / or x pre-filled with NaN or a large
finite value (POISON = none | b | x | bx, POISON_VALUE = nan | big)."""
import os
import sys
import threading

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2407_13997_b200 as w  # noqa: E402
import wrmg_inputs as wi  # noqa: E402

mode = os.environ.get("POISON", "none")
val = float("nan") if os.environ.get("POISON_VALUE", "nan") == "nan" else 1e30
# junk in the caching allocator's free blocks
junk = [torch.full((1 << 20,), val, dtype=torch.float64, device="cuda:0") for _ in range(8)]
del junk
P, snx, ny, k, q, N, nc = 4, 4, 16, 2, 1, 6, 2
gnx = P * snx
g = w.Context(gnx, ny, 1.0 / ny, degree=k, q=q, nslabs=N, dt=1.0 / N, ncoarse=nc)
gl = g.layout
f = wi.spacetime_field(gl["nnode"], N, q, 9)
bg = g.empty()
g.rhs(torch.as_tensor(f, dtype=torch.float64, device="cuda:0"), bg)
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
        if "b" in mode:
            b.fill_(val)
        cc.rhs(torch.as_tensor(fl.reshape(-1), device="cuda:0"), b)
        xx = cc.empty()
        if "x" in mode:
            xx.fill_(val)
        its[r] = cc.fgmres(b, xx, restart=30, maxit=60, rtol=1e-10)[0]
        st.synchronize()
        cc.close()


th = [threading.Thread(target=rank_fn, args=(r,)) for r in range(P)]
for t in th:
    t.start()
for t in th:
    t.join()
hub.close()
print(f"POISON={mode}/{os.environ.get('POISON_VALUE', 'nan')} guard={os.environ.get('WRMG_GUARD')}: strips its {its} vs one rank {its_g}", flush=True)
