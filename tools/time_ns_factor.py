"""Times one Navier-Stokes linearisation (assembly + block inversion, H1/H4/H5) at the
C3 discretisation (P2-P1 x DG1, 64^2, N = 64, Re 100, wind state) or, with --c4, at
C4's P3-P2 x DG1 on 128^2 with --slabs slabs; prints the per-kernel device times.
The inversion kernel is chosen by the library's WRMG_NS_FACTOR_* environment."""
import argparse
import json
import sys

import torch

sys.path.insert(0, ".")
import paper_2407_13997_b200 as w  # noqa: E402
import wrmg_inputs as wi  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--c4", action="store_true")
ap.add_argument("--slabs", type=int, default=None)
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
n, k, q, N, R = (128, 2, 1, a.slabs or 8, 1000.0) if a.c4 else (64, 1, 1, a.slabs or 64, 100.0)
dt = 1.0 / N
c = w.Context(n, n, 1.0 / n, degree=k, q=q, nslabs=N, dt=dt, problem="ns", reynolds=R, bc="lid", omega_mg=0.8)
W = torch.as_tensor(wi.wind_state(n, n, 1.0 / n, k, N, q, dt), device="cuda:0")
c.linearize(W)
torch.cuda.synchronize()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
c.profile(True)
ev[0].record()
for _ in range(a.reps):
    c.linearize(W)
ev[1].record()
torch.cuda.synchronize()
st = {f"{x}@L{l}": round(v["ms"] / a.reps, 3) for (x, l), v in sorted(c.kernel_stats().items(), key=lambda kv: -kv[1]["ms"])}
c.profile(False)
print(json.dumps({"linearize_ms": ev[0].elapsed_time(ev[1]) / a.reps, "kernels_ms": st}))
