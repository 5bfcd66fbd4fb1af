"""C2 solve time with and without the library's per-launch profiling events, and the
summed kernel time: how much of the step is launch / host-sync idle."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2407_13997_b200 as w  # noqa: E402

n, k, q, N = 128, 3, 1, 128
ctx = w.Context(n, n, 1.0 / n, degree=k, q=q, nslabs=N, dt=1.0 / N, kappa=1.0)
fhat = ctx.empty()
ctx.fill_uniform(fhat, first_id=0, seed=0)
b = ctx.empty()
ctx.rhs(fhat, b)
x = ctx.empty()
solve = lambda: ctx.fgmres(b, x, restart=30, maxit=200, rtol=1e-8)
for _ in range(3):
    solve()
torch.cuda.synchronize()
for prof in (False, True, False, True):
    ctx.profile(prof)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        solve()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    kms = sum(s["ms"] for s in ctx.kernel_stats().values()) / 5 if prof else float("nan")
    ctx.profile(False)
    print(f"profile={prof}: {ms:.3f} ms/solve, kernel sum {kms:.3f} ms")
