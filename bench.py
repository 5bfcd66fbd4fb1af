#!/usr/bin/env python
"""Benchmark of the WRMG hot path on B200 (contract: see DESIGN.md "Measurement").

Workload (N=1): BASELINE.json configs[1] (C2): heat equation on the unit square,
128x128 anti-diagonal mesh, P3 in space, DG1 in time, 128 slabs, dt = 1/128,
kappa = 1, Dirichlet 0, f = seeded U[-1,1] nodal coefficients (R6);
FGMRES(30) preconditioned by WRMG V(1,1) to 1e-8 relative residual, FP64.

One step = one complete FGMRES-WRMG solve from x0 = 0 (every residual,
smoother sweep on every level, restriction, prolongation, coarse solve and
Krylov step of the solve).  metric value = smoother space-time DoF updates in
the step (iterations x sum over smoothed levels of free DoFs x (nu_pre+nu_post))
divided by the step time.  Vectors are 303 MB > 126 MB L2, so no L2 flush is
needed between steps.

--impl reference times the CPU oracle (oracle/, the only other place bench.py
executes it) on a bounded sample of the same workload.
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "WR patch-smoother space-time DOF updates/s (FP64)"
UNIT = "DoF-updates/s"
CFG = dict(n=128, k=3, q=1, N=128, kappa=1.0, restart=30, rtol=1e-8)


def peaks():
    p = {}
    try:
        p = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    hbm = p.get("hbm_gbs")
    hbm_src = "measured (MEASURED_PEAKS.json hbm_gbs)"
    if not hbm:
        hbm, hbm_src = 6650.0, "fallback (B200_PROFILING.md)"
    # FP64: no measured entry; derived from unit counts and clocks:
    # 148 SMs x 64 FP64 FMA/clk x 2 flop x 1.965 GHz
    fp64 = 148 * 64 * 2 * 1.965e9 / 1e12
    return hbm, hbm_src, fp64


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms (B200_PROFILING.md)."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def dist_setup(args):
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if ws > 1:
        import torch.distributed as dist
        import torch
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    return ws, rank, local


def max_over_ranks(x, ws):
    if ws == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(ws):
    if ws > 1:
        import torch.distributed as dist
        dist.barrier()


def ncu_traffic(kclass, path=None, names=None):
    """dram__bytes_read.sum + dram__bytes_write.sum of the finest-level launch of
    the kernel behind a timing class, from a committed `ncu --set full` summary
    (default: the C2 bench's profiles/r01_final_c2_ncu.txt); (None, None) if absent."""
    import re
    names = names or {"residual": "k_residual_mac", "sweep": "k_sweep_sym", "krylov": "k_krylov"}
    path = path or os.path.join(ROOT, "profiles", "r02_c2_ncu.txt")
    if kclass not in names or not os.path.exists(path):
        return None, None
    best = None
    for block in open(path).read().split("## ")[1:]:
        if names[kclass] not in block.splitlines()[0]:
            continue
        vals = {}
        for key in ("gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum"):
            m = re.search(key + r"\s+([0-9.]+)\s+(\w+)", block)
            if m:
                scale = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0, "us": 1.0, "ms": 1e3}.get(m.group(2), 1.0)
                vals[key] = float(m.group(1)) * scale
        if len(vals) == 3 and (best is None or vals["gpu__time_duration.sum"] > best[0]):
            best = (vals["gpu__time_duration.sum"], vals["dram__bytes_read.sum"] + vals["dram__bytes_write.sum"])
    if best is None:
        return None, None
    return best[1], os.path.relpath(path, ROOT) + " (ncu --set full, finest-level launch)"


# --------------------------------------------------------------------- oracle
def oracle_sample(n, N, repeats=1):
    """Time the oracle (as it stands) on a bounded sample: the C2 discretisation
    (P3 x DG1, kappa 1, FGMRES(30) + V(1,1) to 1e-8) on an n x n mesh with N slabs,
    single host thread.  Returns (DoF-updates/s, seconds per solve, iterations)."""
    from threadpoolctl import threadpool_limits

    import wrmg_inputs as wi
    from oracle import krylov, multigrid
    with threadpool_limits(1):
        H = multigrid.Hierarchy(n, n, 1.0 / n, CFG["k"], CFG["q"], N, 1.0 / N, kappa=CFG["kappa"])
        p = H.fine
        b = p.rhs(wi.spacetime_field(p.nnode, N, CFG["q"], 0))
        upd_vc = sum(int(L.prob.free.sum()) * L.prob.NT * 2 for L in H.levels[1:])
        times, its = [], 0
        for _ in range(repeats):
            t0 = time.perf_counter()
            x, its, hist, st = krylov.fgmres(lambda v: p.A @ v, lambda r: multigrid.vcycle(H, r), b,
                                             restart=CFG["restart"], rtol=CFG["rtol"])
            times.append(time.perf_counter() - t0)
    t = statistics.median(times)
    return its * upd_vc / t, t, its, H, b, upd_vc


def run_reference(args, ws, rank):
    if rank != 0:
        return
    import numpy as np  # noqa: F401
    from threadpoolctl import threadpool_limits

    from oracle import krylov, multigrid
    n, N = 16, 32
    import wrmg_inputs as wi
    with threadpool_limits(1):
        H = multigrid.Hierarchy(n, n, 1.0 / n, CFG["k"], CFG["q"], N, 1.0 / N, kappa=CFG["kappa"])
        p = H.fine
        b = p.rhs(wi.spacetime_field(p.nnode, N, CFG["q"], 0))
        upd_vc = sum(int(L.prob.free.sum()) * L.prob.NT * 2 for L in H.levels[1:])
        solve = lambda: krylov.fgmres(lambda v: p.A @ v, lambda r: multigrid.vcycle(H, r), b,
                                      restart=CFG["restart"], rtol=CFG["rtol"])
        for _ in range(args.warmup):
            solve()
        t0 = time.perf_counter()
        tot = 0
        for _ in range(args.steps):
            x, its, hist, st = solve()
            tot += its * upd_vc
        el = time.perf_counter() - t0
    v = tot / el
    sample = (f"oracle FGMRES(30)+V(1,1) solve to 1e-8 of the C2 discretisation (P3 x DG1, kappa 1) on a "
              f"{n}x{n} mesh with N={N} slabs per step, 1 host thread")
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * el / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": "C2 (BASELINE configs[1]) bounded oracle sample", "mesh": n, "degree": 3,
                       "q": 1, "nslabs": N},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": 1, "kind": "oracle", "sample": sample},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------- GPU arm
def top_roofline(stats, ncu_path=None, ncu_names=None):
    """Roofline object for the timing class with the largest device time (C3, C5
    lines): achieved algorithmic bytes (or flops) per launch over its measured
    per-launch time, against the measured HBM peak or the derived FP64 peak,
    whichever bounds it."""
    hbm, hbm_src, fp64 = peaks()
    tot = sum(s["ms"] for s in stats.values())
    (a, l), st = max(stats.items(), key=lambda kv: kv[1]["ms"])
    t = st["ms"] / st["launches"] / 1e3
    gbs, tfs = st["bytes"] / st["launches"] / t / 1e9, st["flops"] / st["launches"] / t / 1e12
    alu = st["flops"] / (fp64 * 1e12) > st["bytes"] / (hbm * 1e9)
    traffic, src = (None, None)
    if ncu_path:
        traffic, src = ncu_traffic(a, os.path.join(ROOT, "profiles", ncu_path), ncu_names)
    return {"bound": "alu" if alu else "hbm", "achieved": tfs if alu else gbs,
            "peak": fp64 if alu else hbm, "unit": "TFLOP/s" if alu else "GB/s",
            "frac": (tfs / fp64) if alu else (gbs / hbm), "traffic": traffic, "traffic_source": src,
            "kernel": f"{a}@L{l}",
            "share_of_kernel_time": st["ms"] / tot if tot else None,
            "peak_source": hbm_src if not alu else "derived: 148 SM x 64 FP64 FMA/clk x 2 x 1.965 GHz"}


def run_c5(args, ws, rank, local):
    """BASELINE configs[4] (C5), per GPU (weak reading R24): heat, P2 x DG1,
    N = 256 (dt = 1/256, T = 1), 1024x1024 mesh, 20 stationary V(1,1) cycles
    u <- u + V(b - A u) from u = 0 (one step = the 20 cycles)."""
    import torch

    import paper_2407_13997_b200 as w
    torch.cuda.set_device(local)
    n, k, q, N = args.c5_n, 2, 1, 256
    stream = torch.cuda.current_stream()
    t0 = time.time()
    kw = {}
    if ws > 1:  # weak reading R24: [0, ws] x [0, 1], 1024 x 1024 cells per GPU, strips with NCCL halos
        import torch.distributed as dist
        idt = torch.zeros(128, dtype=torch.uint8, device=f"cuda:{local}")
        if rank == 0:
            idt.copy_(torch.frombuffer(bytearray(w.nccl_unique_id()), dtype=torch.uint8))
        dist.broadcast(idt, 0)
        kw = dict(rank=rank, nranks=ws, nccl_id=bytes(idt.cpu().numpy().tobytes()))
    ctx = w.Context(ws * n, n, 1.0 / n, degree=k, q=q, nslabs=N, dt=1.0 / N, device=local, stream=stream.cuda_stream,
                    **kw)
    setup_s = time.time() - t0
    lay = ctx.layout
    fhat = ctx.empty()
    NT = lay["nt"]
    GLx = k * ws * n + 1
    if ws == 1:
        ctx.fill_uniform(fhat, 0, 0)
    else:  # R6 at global canonical ids: local row J holds global columns g0 .. g0 + lx - 1
        fv = fhat.view(lay["ly"], lay["lx"] * NT)
        for J in range(lay["ly"]):
            ctx.fill_uniform(fv[J], (J * GLx + lay["g0"]) * NT, 0)
    b = ctx.empty()
    ctx.rhs(fhat, b)
    del fhat
    u, r, z = ctx.empty(), ctx.empty(), ctx.empty()
    upd = lay["smooth_dof_updates_per_vcycle"]
    upd_all = ws * upd
    if ws > 1:
        import torch.distributed as dist
        tu = torch.tensor([float(upd)], dtype=torch.float64, device=f"cuda:{local}")
        dist.all_reduce(tu)
        upd_all = tu.item()

    def owned_sq(v):
        a = v.view(lay["ly"], lay["lx"], NT)[:, lay["own0"]:lay["own1"] + 1, :]
        t = (a * a).sum().reshape(1)
        if ws > 1:
            import torch.distributed as dist
            dist.all_reduce(t)
        return float(t.item())

    def step():
        u.zero_()
        ctx.stationary(b, u, 20)  # 20 x (u <- u + V(b - A u)), every operation in the library

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    ctx.profile(True)
    l0 = w.launch_count()
    barrier(ws)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize()
    barrier(ws)
    ms = max_over_ranks(e0.elapsed_time(e1), ws)
    stats = ctx.kernel_stats()
    clk = clocks.stop()
    ctx.residual(u, b, r)
    rel = (owned_sq(r) / owned_sq(b)) ** 0.5
    per_kernel = {f"{a}@L{l}": {"launches": s["launches"], "ms": round(s["ms"], 3),
                                "GBs": round(s["bytes"] / (s["ms"] / 1e3) / 1e9, 1) if s["ms"] > 0 else None,
                                "TFs": round(s["flops"] / (s["ms"] / 1e3) / 1e12, 3) if s["ms"] > 0 else None}
                  for (a, l), s in sorted(stats.items(), key=lambda kv: -kv[1]["ms"])}
    line = {"metric": METRIC, "value": 20 * upd_all * args.steps / (ms / 1e3), "unit": UNIT, "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"C5 = BASELINE configs[4] per GPU (weak, R24): heat P2 x DG1, N=256, "
                                   f"{n}x{n} cells per GPU, global [0,{ws}]x[0,1], 20 V(1,1)",
                       "ndof_per_gpu": lay["ndof"], "levels": lay["nlevels"], "setup_s": round(setup_s, 2),
                       "parallelism": f"{ws} spatial strips, NCCL halo per operator" if ws > 1 else "1 GPU",
                       "l2": "inputs larger than L2 (17 GB vectors); no flush"},
            "relres_after_20_vcycles": rel, "roofline": top_roofline(stats), "per_kernel": per_kernel, "clocks": clk,
            "gpu_launches": w.launch_count() - l0}
    if rank == 0:
        print(json.dumps(line), flush=True)
    ctx.close()


def run_c3(args, ws, rank, local):
    """BASELINE configs[2] (C3): Oseen = one Newton linearisation of Navier-Stokes
    (R18) at the wind w = curl psi, P2-P1 Taylor-Hood x DG1, 64x64, N = 64, T = 1
    (R21), Re = 100, lid BCs, b ~ U[-1,1) on free rows (R6); omega_mg = 0.8
    (R-omega-NS).  One step = the C3 protocol of SURVEY 8(d) with fixed work:
    10 smoother sweeps (omega = 1), one V(1,1) on the residual, and one FGMRES(30)
    restart cycle (30 preconditioned iterations); the additive Vanka V(1,1) does not
    contract on this wind at Re = 100 (NS findings; the oracle agrees), so
    a solve-to-tolerance step would not terminate.  The linearisation (assembly +
    batched block inversion, H1/H4/H5) is timed apart."""
    import numpy as np
    import torch

    import paper_2407_13997_b200 as w
    import wrmg_inputs as wi
    torch.cuda.set_device(local)
    n, k, q, N, R, T = 64, 1, 1, 64, 100.0, 1.0
    dt = T / N
    stream = torch.cuda.current_stream()
    kw = strip_kwargs(ws, rank, local)
    t0 = time.time()
    ctx = w.Context(n, n, 1.0 / n, degree=k, q=q, nslabs=N, dt=dt, problem="ns", reynolds=R, bc="lid",
                    omega_mg=0.8, device=local, stream=stream.cuda_stream, **kw)
    setup_s = time.time() - t0
    lay = ctx.layout
    Wg = wi.wind_state(n, n, 1.0 / n, k, N, q, dt)
    if ws > 1:  # this strip's window of the global state (the library refreshes non-owned columns itself)
        Wg = ns_window(Wg, lay, (k + 1) * n + 1, (k + 1) * n + 1, k * n + 1, k * n + 1, lay["nt"])
    W = torch.as_tensor(Wg, device=f"cuda:{local}")
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ctx.linearize(W)  # warm
    torch.cuda.synchronize()
    ctx.profile(True)
    barrier(ws)
    ev[0].record(stream)
    ctx.linearize(W)
    ev[1].record(stream)
    torch.cuda.synchronize()
    lin_ms = max_over_ranks(ev[0].elapsed_time(ev[1]), ws)
    lin_stats = {f"{a}@L{l}": {"ms": round(v["ms"], 3), "TFs": round(v["flops"] / (v["ms"] / 1e3) / 1e12, 3)}
                 for (a, l), v in ctx.kernel_stats().items()}
    ctx.profile(False)
    f = ns_fill_canonical(ctx, k, n)
    b = ctx.empty()
    ctx.rhs(f, b)
    x = ctx.empty()
    u, r, z = ctx.empty(), ctx.empty(), ctx.empty()
    upd_vc = sum_over_ranks(lay["smooth_dof_updates_per_vcycle"], ws, local)
    upd_sweep = sum_over_ranks(lay["nfree_owned_st"], ws, local)

    def solve():
        u.zero_()
        ctx.smooth(u, b, 10, 1.0)
        ctx.residual(u, b, r)
        ctx.vcycle(r, z)
        its, rel, st = ctx.fgmres(b, x, restart=30, maxit=30, rtol=1e-8)
        return its, rel, st

    for _ in range(args.warmup):
        solve()
    torch.cuda.synchronize()
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    ctx.profile(True)
    l0 = w.launch_count()
    barrier(ws)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    tot, its_l, st_l = 0, [], []
    for _ in range(args.steps):
        its, rel, st = solve()
        tot += 10 * upd_sweep + (1 + its) * upd_vc
        its_l.append(its)
        st_l.append((st, rel))
    e1.record(stream)
    torch.cuda.synchronize()
    barrier(ws)
    ms = max_over_ranks(e0.elapsed_time(e1), ws)
    stats = ctx.kernel_stats()
    ctx.profile(False)
    clk = clocks.stop()
    z = ctx.empty()
    ev2 = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    ev2[0].record(stream)
    for _ in range(5):
        ctx.vcycle(b, z)
    ev2[1].record(stream)
    u = ctx.zeros()
    ev2[2].record(stream)
    for _ in range(5):
        ctx.smooth(u, b, 1, 1.0)
    ev2[3].record(stream)
    torch.cuda.synchronize()
    per_kernel = {f"{a}@L{l}": {"launches": s["launches"], "ms": round(s["ms"], 3),
                                "GBs": round(s["bytes"] / (s["ms"] / 1e3) / 1e9, 1) if s["ms"] > 0 else None,
                                "TFs": round(s["flops"] / (s["ms"] / 1e3) / 1e12, 3) if s["ms"] > 0 else None}
                  for (a, l), s in sorted(stats.items(), key=lambda kv: -kv[1]["ms"])}
    line = {"metric": METRIC, "value": tot / (ms / 1e3), "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
            "scaling": "strong" if ws > 1 else "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": "C3 = BASELINE configs[2]: Oseen (Newton Jacobian at w = curl psi), P2-P1 x DG1, "
                                   "64x64, N=64, T=1, Re=100, lid; step = 10 sweeps + V(1,1) + 30 FGMRES(30) "
                                   "iterations, omega_mg 0.8",
                       "parallelism": f"{ws} spatial strips, NCCL halos" if ws > 1 else "1 GPU",
                       "ndof": lay["ndof"], "nfree_st": lay["nfree_st"], "levels": lay["nlevels"],
                       "npatch": lay["npatch"], "mp_max": lay["mp_max"], "setup_s": round(setup_s, 2)},
            "fgmres_iterations": its_l[0], "fgmres_status_relres": st_l[0], "linearize_ms": lin_ms,
            "linearize_kernels": lin_stats,
            "vcycle_ms": ev2[0].elapsed_time(ev2[1]) / 5, "smoother_sweep_ms": ev2[2].elapsed_time(ev2[3]) / 5,
            "roofline": top_roofline(stats, "r01_final_c3_ncu.txt",
                                     {"sweep": "k_ns_sweep", "residual": "k_ns_residual"}),
            "per_kernel": per_kernel, "clocks": clk, "gpu_launches": w.launch_count() - l0}
    if rank == 0:
        print(json.dumps(line), flush=True)
    ctx.close()


def strip_kwargs(ws, rank, local):
    """Context kwargs of this rank's spatial strip (NCCL transport; rank 0 draws the id)."""
    if ws == 1:
        return {}
    import torch
    import torch.distributed as dist

    import paper_2407_13997_b200 as w
    idt = torch.zeros(128, dtype=torch.uint8, device=f"cuda:{local}")
    if rank == 0:
        idt.copy_(torch.frombuffer(bytearray(w.nccl_unique_id()), dtype=torch.uint8))
    dist.broadcast(idt, 0)
    return dict(rank=rank, nranks=ws, nccl_id=bytes(idt.cpu().numpy().tobytes()))


def sum_over_ranks(x, ws, local):
    if ws == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(x)], dtype=torch.float64, device=f"cuda:{local}")
    dist.all_reduce(t)
    return t.item()


def ns_fill_canonical(ctx, k, n, seed=0):
    """R6 draws of a Navier-Stokes vector at the GLOBAL canonical ids (sid NT + t): one
    call on one rank; on a strip, per local lattice row of each field (u_x, u_y, p)."""
    lay = ctx.layout
    f = ctx.empty()
    if lay["g0"] == 0 and lay["own1"] == lay["lx"] - 1:
        ctx.fill_uniform(f, 0, seed)
        return f
    NT, Lx, Ly = lay["nt"], lay["lx"], lay["ly"]
    GLux = (k + 1) * n + 1
    GLu = GLux * Ly
    fv = f.view(-1, NT)
    for off, lx, ly, gx, gc0, goff in ((0, Lx, Ly, GLux, lay["g0"], 0), (lay["lu"], Lx, Ly, GLux, lay["g0"], GLu),
                                       (2 * lay["lu"], lay["lpx"], lay["lpy"], k * n + 1, lay["g0p"], 2 * GLu)):
        for J in range(ly):
            ctx.fill_uniform(fv[off + J * lx:off + (J + 1) * lx].reshape(-1), (goff + J * gx + gc0) * NT, seed)
    return f


def ns_window(vg, lay, ly_g, lx_g, lpy_g, lpx_g, NT):
    """This rank's local window (every local column) of a global NS vector (host numpy)."""
    import numpy as np
    lu_g = lx_g * ly_g
    a = vg.reshape(-1, NT)
    gu, gv = a[:lu_g].reshape(ly_g, lx_g, NT), a[lu_g:2 * lu_g].reshape(ly_g, lx_g, NT)
    gp = a[2 * lu_g:].reshape(lpy_g, lpx_g, NT)
    c0, c0p = lay["g0"], lay["g0p"]
    return np.concatenate([gu[:, c0:c0 + lay["lx"]].reshape(-1), gv[:, c0:c0 + lay["lx"]].reshape(-1),
                           gp[:, c0p:c0p + lay["lpx"]].reshape(-1)])


def run_c4(args, ws, rank, local):
    """BASELINE configs[3] (C4): Navier-Stokes lid-driven cavity, P3-P2 Taylor-Hood x
    DG1, 128x128 mesh, dt = 1/128, Re = 1000, linearised at the zero state + lid lift
    (the first Newton step, R26).  The stored (patch, slab) block inverses of the full
    128-slab horizon are 447 GB: one B200 holds N = 32 slabs; with ws > 1
    the mesh is split into ws spatial strips (NCCL halos) and the
    default horizon is N = min(128, 32 ws) -- the full C4 horizon from 4 GPUs on.
    Step = fixed work: 10 Vanka+star sweeps (omega 1) + one residual + one V(1,1) on a
    seeded RHS (omega_mg 0.8); the linearisation (assembly + batched block inversion on
    every level) is timed apart."""
    import torch

    import paper_2407_13997_b200 as w
    torch.cuda.set_device(local)
    n, k, q, R = 128, 2, 1, 1000.0
    N = args.c4_n if args.c4_n else min(128, 32 * ws)
    dt = 1.0 / 128
    stream = torch.cuda.current_stream()
    kw = strip_kwargs(ws, rank, local)
    t0 = time.time()
    ctx = w.Context(n, n, 1.0 / n, degree=k, q=q, nslabs=N, dt=dt, problem="ns", reynolds=R, bc="lid",
                    omega_mg=0.8, device=local, stream=stream.cuda_stream, **kw)
    setup_s = time.time() - t0
    lay = ctx.layout
    NT = lay["nt"]
    Lx, Ly, g0 = lay["lx"], lay["ly"], lay["g0"]
    GLux = (k + 1) * n + 1
    W = torch.zeros(lay["ndof"], dtype=torch.float64, device=f"cuda:{local}")
    top = W.view(-1, NT)[(Ly - 1) * Lx:Ly * Lx]  # u_x on the lid row (local columns), corners excluded
    lo, hi = max(0, 1 - g0), min(Lx, GLux - 1 - g0)
    top[lo:hi].fill_(1.0)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ctx.profile(True)
    barrier(ws)
    ev[0].record(stream)
    ctx.linearize(W)
    ev[1].record(stream)
    torch.cuda.synchronize()
    lin_ms = max_over_ranks(ev[0].elapsed_time(ev[1]), ws)
    lin_stats = {f"{a}@L{l}": {"ms": round(v["ms"], 3), "TFs": round(v["flops"] / (v["ms"] / 1e3) / 1e12, 3)}
                 for (a, l), v in ctx.kernel_stats().items()}
    ctx.profile(False)
    f = ns_fill_canonical(ctx, k, n)
    b = ctx.empty()
    ctx.rhs(f, b)
    del f
    u, r, z = ctx.empty(), ctx.empty(), ctx.empty()
    upd_vc = sum_over_ranks(lay["smooth_dof_updates_per_vcycle"], ws, local)
    upd_sweep = sum_over_ranks(lay["nfree_owned_st"], ws, local)

    def step():
        u.zero_()
        ctx.smooth(u, b, 10, 1.0)
        ctx.residual(u, b, r)
        ctx.vcycle(r, z)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    ctx.profile(True)
    l0 = w.launch_count()
    barrier(ws)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize()
    barrier(ws)
    ms = max_over_ranks(e0.elapsed_time(e1), ws)
    stats = ctx.kernel_stats()
    ctx.profile(False)
    clk = clocks.stop()
    per_kernel = {f"{a}@L{l}": {"launches": s["launches"], "ms": round(s["ms"], 3),
                                "GBs": round(s["bytes"] / (s["ms"] / 1e3) / 1e9, 1) if s["ms"] > 0 else None,
                                "TFs": round(s["flops"] / (s["ms"] / 1e3) / 1e12, 3) if s["ms"] > 0 else None}
                  for (a, l), s in sorted(stats.items(), key=lambda kv: -kv[1]["ms"])}
    tot = args.steps * (10 * upd_sweep + upd_vc)
    full = N == 128
    line = {"metric": METRIC, "value": tot / (ms / 1e3), "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
            "scaling": "weak" if N == 32 * ws else "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": f"C4 = BASELINE configs[3]: NS cavity P3-P2 x DG1, 128x128, dt=1/128, Re=1000, "
                                   f"linearised at the lid lift; N={N} slabs"
                                   + ((" (the full horizon [0, 1]; 447 GB of block inverses: levels whose store "
                                       "does not fit keep a slab window and recompute it in every sweep)")
                                      if full and 32 * ws < 128 else " (the full horizon [0, 1])" if full else
                                      " (--c4-n 128: the full horizon, windowed inverses on one GPU)")
                                   + "; step = 10 sweeps + residual + V(1,1)",
                       "parallelism": f"{ws} spatial strips, NCCL halos" if ws > 1 else "1 GPU",
                       "ndof": lay["ndof"], "nfree_st": lay["nfree_st"], "levels": lay["nlevels"],
                       "npatch": lay["npatch"], "mp_max": lay["mp_max"], "setup_s": round(setup_s, 2)},
            "linearize_ms": lin_ms, "linearize_kernels": lin_stats,
            "roofline": top_roofline(stats), "per_kernel": per_kernel, "clocks": clk,
            "gpu_launches": w.launch_count() - l0}
    if rank == 0:
        print(json.dumps(line), flush=True)
    ctx.close()


def run_gpu(args, ws, rank, local):
    import torch

    import paper_2407_13997_b200 as w
    torch.cuda.set_device(local)
    dev = f"cuda:{local}"
    n, k, q, N = CFG["n"], CFG["k"], CFG["q"], CFG["N"]
    stream = torch.cuda.current_stream()
    kw = {}
    if ws > 1:  # strong scaling: the C2 problem split into ws spatial strips (NCCL halos)
        import torch.distributed as dist
        idt = torch.zeros(128, dtype=torch.uint8, device=dev)
        if rank == 0:
            idt.copy_(torch.frombuffer(bytearray(w.nccl_unique_id()), dtype=torch.uint8))
        dist.broadcast(idt, 0)
        kw = dict(rank=rank, nranks=ws, nccl_id=bytes(idt.cpu().numpy().tobytes()))
    ctx = w.Context(n, n, 1.0 / n, degree=k, q=q, nslabs=N, dt=1.0 / N, kappa=CFG["kappa"], device=local,
                    stream=stream.cuda_stream, scatter=args.scatter, **kw)
    lay = ctx.layout
    ndof = lay["ndof"]
    fhat = ctx.empty()
    if ws == 1:
        ctx.fill_uniform(fhat, first_id=0, seed=0)  # R6 generator at canonical ids
    else:  # R6 at global canonical ids: local row J holds global columns g0 .. g0 + lx - 1
        NT, GLx = lay["nt"], k * n + 1
        fv = fhat.view(lay["ly"], lay["lx"] * NT)
        for J in range(lay["ly"]):
            ctx.fill_uniform(fv[J], (J * GLx + lay["g0"]) * NT, 0)
    b = ctx.empty()
    ctx.rhs(fhat, b)
    del fhat
    x = ctx.empty()
    upd_vc = lay["smooth_dof_updates_per_vcycle"]  # strips: owned rows (+ the replicated levels on rank 0)
    if ws > 1:
        import torch.distributed as dist
        tu = torch.tensor([float(upd_vc)], dtype=torch.float64, device=dev)
        dist.all_reduce(tu)
        upd_vc = tu.item()

    def solve():
        its, rel, st = ctx.fgmres(b, x, restart=CFG["restart"], maxit=200, rtol=CFG["rtol"])
        if st != "WRMG_OK":
            raise RuntimeError(f"FGMRES status {st}")
        return its, rel

    for _ in range(max(args.warmup, 0)):
        solve()
    torch.cuda.synchronize()
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    launches0 = w.launch_count()  # launches before the timed region (ncu -s for the launch list)
    barrier(ws)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    tot_upd, its_list, rels = 0, [], []
    for i in range(args.steps):
        # per-kernel CUDA events on the library's stream during the LAST timed step only: the event
        # pairs around ~300 launches per solve open ~1.35 ms of launch gaps (tools/c2_overhead.py)
        if i == args.steps - 1:
            ctx.profile(True)
        its, rel = solve()
        tot_upd += its * upd_vc
        its_list.append(its)
        rels.append(rel)
    e1.record(stream)
    torch.cuda.synchronize()
    barrier(ws)
    ms_total = e0.elapsed_time(e1)
    launches = w.launch_count() - launches0
    stats = ctx.kernel_stats()
    ctx.profile(False)
    clk = clocks.stop()
    ms_total = max_over_ranks(ms_total, ws)
    ms_step = ms_total / args.steps
    value = tot_upd / (ms_total / 1e3)  # upd_vc already sums the ranks' owned updates

    # dominant kernel (largest device-time share in the timed region)
    hbm, hbm_src, fp64 = peaks()
    tot_ms = sum(s["ms"] for s in stats.values())
    (kname, klvl), ks = max(stats.items(), key=lambda kv: kv[1]["ms"])
    per_launch_ms = ks["ms"] / ks["launches"]
    t_hbm = ks["bytes"] / ks["launches"] / (hbm * 1e9)
    t_fp = ks["flops"] / ks["launches"] / (fp64 * 1e12)
    if t_fp > t_hbm:
        roof = {"bound": "alu", "achieved": ks["flops"] / ks["launches"] / (per_launch_ms / 1e3) / 1e12,
                "peak": fp64, "unit": "TFLOP/s"}
    else:
        roof = {"bound": "hbm", "achieved": ks["bytes"] / ks["launches"] / (per_launch_ms / 1e3) / 1e9,
                "peak": hbm, "unit": "GB/s"}
    roof["frac"] = roof["achieved"] / roof["peak"]
    roof["traffic"], roof["traffic_source"] = ncu_traffic(kname)
    roof["kernel"] = f"{kname} (level {klvl} of {lay['nlevels']}, finest = {lay['nlevels'] - 1})"
    roof["share_of_kernel_time"] = ks["ms"] / tot_ms if tot_ms else None
    roof["peak_source"] = (hbm_src if roof["bound"] == "hbm" else
                           "derived: 148 SM x 64 FP64 FMA/clk x 2 x 1.965 GHz (no measured FP64 peak)")
    roof["hbm_achieved_GBs"] = ks["bytes"] / ks["launches"] / (per_launch_ms / 1e3) / 1e9
    roof["fp64_achieved_TFs"] = ks["flops"] / ks["launches"] / (per_launch_ms / 1e3) / 1e12
    # the three largest timing classes against their own binding roof (context for the headline kernel)
    roof_top = []
    for (a, l), st in sorted(stats.items(), key=lambda kv: -kv[1]["ms"])[:3]:
        t_ms = st["ms"] / st["launches"]
        gbs = st["bytes"] / st["launches"] / (t_ms / 1e3) / 1e9
        tfs = st["flops"] / st["launches"] / (t_ms / 1e3) / 1e12
        alu = st["flops"] / (fp64 * 1e12) > st["bytes"] / (hbm * 1e9)
        roof_top.append({"kernel": f"{a}@L{l}", "bound": "alu" if alu else "hbm",
                         "achieved": tfs if alu else gbs, "unit": "TFLOP/s" if alu else "GB/s",
                         "peak": fp64 if alu else hbm, "frac": (tfs / fp64) if alu else (gbs / hbm),
                         "share_of_kernel_time": st["ms"] / tot_ms if tot_ms else None})
    roof["top_kernels"] = roof_top
    # the heat sweep's binding resource is the L2's FP64 atomic rate of its weighted additive
    # scatter: one update per (patch DoF, time value), against the rate
    # tools/atomic_probe.cu measured for contiguous lanes on this B200 (profiles/r02_atomic_probe.txt)
    if args.scatter == "atomic" and ws == 1:
        _, psz = w.wrmg_plan_patches(n, n, 1.0 / n, k)
        upd = float(psz.sum()) * (q + 1) * N
        sw = stats.get(("sweep", lay["nlevels"] - 1))
        if sw and sw["launches"]:
            t_l = sw["ms"] / sw["launches"] / 1e3
            roof["sweep_l2_atomic"] = {"kernel": f"sweep@L{lay['nlevels'] - 1}", "bound": "l2_fp64_atomics",
                                       "updates_per_launch": upd, "achieved": upd / t_l / 1e9, "peak": 320.3,
                                       "unit": "G element-updates/s", "frac": upd / t_l / 1e9 / 320.3,
                                       "peak_source": "measured: tools/atomic_probe.cu, contiguous red.global.add.f64"}
    per_kernel = {f"{a}@L{l}": {"launches": s["launches"], "ms": round(s["ms"], 4),
                                "GBs": round(s["bytes"] / (s["ms"] / 1e3) / 1e9, 1) if s["ms"] > 0 else None,
                                "TFs": round(s["flops"] / (s["ms"] / 1e3) / 1e12, 3) if s["ms"] > 0 else None}
                  for (a, l), s in sorted(stats.items(), key=lambda kv: -kv[1]["ms"])}

    # V-cycle time and finest-level smoother sweep throughput (separately timed)
    r = ctx.empty()
    ctx.residual(x, b, r)
    z = ctx.empty()
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    ev[0].record(stream)
    for _ in range(10):
        ctx.vcycle(b, z)
    ev[1].record(stream)
    u = ctx.zeros()
    ev[2].record(stream)
    for _ in range(10):
        ctx.smooth(u, b, 1, 1.0)
    ev[3].record(stream)
    torch.cuda.synchronize()
    vcycle_ms = ev[0].elapsed_time(ev[1]) / 10
    sweep_ms = ev[2].elapsed_time(ev[3]) / 10

    # end to end through the public API on HOST buffers: wrmg_fgmres_host solves e2e_steps
    # right-hand sides held in pinned host memory, each uploaded, solved and downloaded by the
    # library (the upload of rhs i+1 and the download of x i-1 on its copy stream during solve i);
    # the timed region spans every copy.
    # a serving loop of max(20, steps) solves over 4 pinned RHS / solution buffers used in turn (the
    # pipeline's fill and drain -- one unhidden upload and download -- amortised over the loop)
    e2e_steps = max(20, args.steps)
    hb4 = [b.detach().cpu().pin_memory() for _ in range(4)]
    hx4 = [torch.empty_like(hb4[0]).pin_memory() for _ in range(4)]
    hb = [hb4[i % 4] for i in range(e2e_steps)]
    hx = [hx4[i % 4] for i in range(e2e_steps)]
    barrier(ws)
    torch.cuda.synchronize()
    ea, eb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ea.record(stream)
    its_h, rel_h, st_h = ctx.fgmres_host(hb, hx, restart=CFG["restart"], maxit=200, rtol=CFG["rtol"])
    eb.record(stream)
    torch.cuda.synchronize()
    if st_h != "WRMG_OK":
        raise RuntimeError(f"FGMRES (host buffers) status {st_h}")
    assert its_h[-1] == its_list[-1], (its_h, its_list)
    e2e_upd = sum(its_h) * upd_vc
    e2e_ms = max_over_ranks(ea.elapsed_time(eb), ws)
    e2e = {"value": e2e_upd / (e2e_ms / 1e3), "unit": UNIT, "h2d_bytes_per_step": ws * ndof * 8,
           "d2h_bytes_per_step": ws * ndof * 8, "steps": e2e_steps,
           "api": "wrmg_fgmres_host (C ABI, host buffers)",
           "pipelining": "inside the library: upload of rhs i+1 and download of x i-1 on a copy stream during solve i"}

    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "strong" if ws > 1 else "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": "C2 = BASELINE configs[1]: heat, unit square 128x128, P3 x DG1, N=128, "
                                   "dt=1/128, kappa=1, Dirichlet 0, f ~ U[-1,1] seed 0; FGMRES(30)+WRMG V(1,1) "
                                   "to 1e-8; one step = one full solve",
                       "ndof": ndof, "nfree_st": lay["nfree_st"], "levels": lay["nlevels"],
                       "parallelism": (f"{ws} spatial strips of the one C2 problem (NCCL halos; levels narrower "
                                       f"than 2 cells per strip replicated)") if ws > 1 else "1 GPU",
                       "l2": "inputs larger than L2 (303 MB vectors vs 126 MB L2); no flush",
                       "scatter": args.scatter},
            "fgmres_iterations": its_list[0], "final_relres": rels[-1],
            "vcycle_ms": vcycle_ms, "smoother_sweep_ms": sweep_ms,
            "smoother_sweep_dof_updates_per_s": lay["nfree_st"] / (sweep_ms / 1e3),
            "roofline": roof, "per_kernel": per_kernel, "per_kernel_steps": 1,
            "per_kernel_note": "kernel times from CUDA events on the library stream during the last timed step",
            "e2e": e2e, "gpu_launches": launches, "clocks": clk, "launches_before_timed": launches0}
    if ws == 1 and rank == 0 and not args.no_cpu_baseline:
        v, t, its, *_ = oracle_sample(16, 128)
        line["cpu_baseline"] = {"value": v, "unit": UNIT, "cores": 1, "kind": "oracle",
                                "sample": f"oracle FGMRES(30)+V(1,1) to 1e-8, C2 discretisation (P3 x DG1, "
                                          f"N=128) on a 16x16 mesh, 1 host thread, {its} iterations in {t:.1f} s"}
    if rank == 0:
        print(json.dumps(line), flush=True)
    ctx.close()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="wrmg", choices=["wrmg", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--config", default="C2", choices=["C2", "C3", "C4", "C5"])
    ap.add_argument("--c4-n", type=int, default=0,
                    help="C4 slabs (0: min(128, 32 x GPUs); one GPU stores the inverses of 32, more slabs "
                         "recompute windows of them in every sweep)")
    ap.add_argument("--c5-n", type=int, default=1024, help="C5 cells per side per GPU (1024 = the config)")
    ap.add_argument("--scatter", default="atomic", choices=["atomic", "colour"],
                    help="weighted additive scatter of the heat sweep (H8): FP64 atomics or coloured passes")
    args = ap.parse_args()
    ws, rank, local = dist_setup(args) if args.impl == "wrmg" else (
        int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")), 0)
    if args.impl == "reference":
        run_reference(args, ws, rank)
        return
    if args.config == "C5":
        run_c5(args, ws, rank, local)
    elif args.config == "C3":
        run_c3(args, ws, rank, local)
    elif args.config == "C4":
        run_c4(args, ws, rank, local)
    else:
        run_gpu(args, ws, rank, local)
    if ws > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
