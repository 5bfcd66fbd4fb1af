"""ctypes marshalling for include/wrmg.h.  Names follow the C ABI."""
import ctypes
import os

import numpy as np

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libwrmg.so")
if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: build it with `make` or __graft_entry__.build(); "
                      "there is no CPU fallback")
lib = ctypes.CDLL(LIB_PATH)

c_i32, c_i64, c_dbl, c_vp = ctypes.c_int32, ctypes.c_int64, ctypes.c_double, ctypes.c_void_p

STATUS = {0: "WRMG_OK", 1: "WRMG_E_INVALID", 2: "WRMG_E_UNSUPPORTED", 3: "WRMG_E_OOM", 4: "WRMG_E_SINGULAR",
          5: "WRMG_E_BREAKDOWN", 6: "WRMG_E_NOT_CONVERGED", 7: "WRMG_E_CUDA", 8: "WRMG_E_NCCL"}


class wrmg_mesh(ctypes.Structure):
    _fields_ = [("gnx", c_i32), ("gny", c_i32), ("x0", c_i32), ("nx", c_i32), ("h", c_dbl), ("ncoarse", c_i32)]


class wrmg_coeffs(ctypes.Structure):
    _fields_ = [("problem", c_i32), ("bc", c_i32), ("kappa", c_dbl), ("reynolds", c_dbl), ("lid_speed", c_dbl),
                ("weights", c_i32), ("omega_mg", c_dbl), ("nu_pre", c_i32), ("nu_post", c_i32),
                ("factor_mode", c_i32), ("device", c_i32), ("stream", c_vp), ("rank", c_i32), ("nranks", c_i32),
                ("nccl_unique_id", c_vp), ("loopback_hub", c_vp), ("smoother", c_i32), ("cheb_steps", c_i32),
                ("cheb_seed", ctypes.c_uint64), ("scatter", c_i32), ("orth", c_i32)]


class wrmg_layout_t(ctypes.Structure):
    _fields_ = [("nnode", c_i64), ("nt", c_i64), ("ndof", c_i64), ("nfree_st", c_i64), ("lx", c_i32),
                ("ly", c_i32), ("nlevels", c_i32), ("degree", c_i32), ("q", c_i32), ("nslabs", c_i32),
                ("npatch", c_i64), ("mp_max", c_i32), ("npatch_types", c_i32),
                ("smooth_dof_updates_per_vcycle", c_i64), ("own0", c_i32), ("own1", c_i32), ("g0", c_i32),
                ("nfree_owned_st", c_i64), ("lu", c_i64), ("lpx", c_i32), ("lpy", c_i32), ("own0p", c_i32),
                ("own1p", c_i32), ("g0p", c_i32)]


class wrmg_kernel_stat(ctypes.Structure):
    _fields_ = [("launches", c_i64), ("ms", c_dbl), ("bytes", c_dbl), ("flops", c_dbl)]


KERNEL_CLASSES = ["residual", "sweep", "restrict", "prolong", "coarse", "krylov", "factor"]

_P = ctypes.POINTER
_sig = {
    "wrmg_setup": (c_i32, [_P(wrmg_mesh), c_i32, c_i32, c_i32, c_dbl, _P(wrmg_coeffs), _P(c_vp)]),
    "wrmg_layout": (c_i32, [c_vp, _P(wrmg_layout_t)]),
    "wrmg_linearize": (c_i32, [c_vp, c_vp]),
    "wrmg_rhs": (c_i32, [c_vp, c_vp, c_vp]),
    "wrmg_rhs_initial": (c_i32, [c_vp, c_vp, c_vp]),
    "wrmg_cheb_lambda": (c_i32, [c_vp, c_i32, _P(c_dbl)]),
    "wrmg_set_boundary_values": (c_i32, [c_vp, c_vp]),
    "wrmg_residual": (c_i32, [c_vp, c_vp, c_vp, c_vp, c_i32]),
    "wrmg_apply": (c_i32, [c_vp, c_vp, c_vp]),
    "wrmg_smooth": (c_i32, [c_vp, c_vp, c_vp, c_i32, c_dbl]),
    "wrmg_vcycle": (c_i32, [c_vp, c_vp, c_vp]),
    "wrmg_restrict": (c_i32, [c_vp, c_i32, c_vp, c_vp]),
    "wrmg_prolong_add": (c_i32, [c_vp, c_i32, c_vp, c_vp]),
    "wrmg_level_size": (c_i32, [c_vp, c_i32, _P(c_i64)]),
    "wrmg_fgmres": (c_i32, [c_vp, c_vp, c_vp, c_i32, c_i32, c_dbl, c_dbl, _P(c_i32), _P(c_dbl)]),
    "wrmg_fgmres_host": (c_i32, [c_vp, c_i32, c_vp, c_vp, c_i32, c_i32, c_dbl, c_dbl, _P(c_i32), _P(c_dbl)]),
    "wrmg_stationary": (c_i32, [c_vp, c_vp, c_vp, c_i32]),
    "wrmg_newton": (c_i32, [c_vp, c_vp, c_dbl, c_i32, _P(c_i32), _P(c_i32)]),
    "wrmg_newton_rhs": (c_i32, [c_vp, c_vp, c_vp, c_dbl, c_i32, _P(c_i32), _P(c_i32)]),
    "wrmg_batched_lu": (c_i32, [c_vp, c_vp, c_i32, c_i32, c_vp, c_vp]),
    "wrmg_fill_uniform": (c_i32, [c_vp, c_vp, c_i64, ctypes.c_uint64, ctypes.c_uint64]),
    "wrmg_sync": (c_i32, [c_vp]),
    "wrmg_last_error": (ctypes.c_char_p, [c_vp, _P(c_i32), _P(c_i32), _P(c_i32)]),
    "wrmg_destroy": (None, [c_vp]),
    "wrmg_plan": (c_i32, [_P(wrmg_mesh), c_i32, c_i32, c_i32, _P(wrmg_layout_t)]),
    "wrmg_plan_patches": (c_i32, [_P(wrmg_mesh), c_i32, c_vp, c_vp]),
    "wrmg_profile": (c_i32, [c_vp, c_i32]),
    "wrmg_kernel_stats": (c_i32, [c_vp, c_vp]),
    "wrmg_launch_count": (c_i64, []),
    "wrmg_guard_violations": (c_i64, []),
    "wrmg_debug_fetch": (c_i32, [c_vp, c_i32, c_i32, c_vp, c_i64]),
    "wrmg_nccl_unique_id": (c_i32, [c_vp]),
    "wrmg_hessenberg_eig": (c_i32, [c_vp, c_i32, c_vp, c_vp]),
    "wrmg_plan_strip": (c_i32, [_P(wrmg_mesh), c_i32, c_i32, c_i32, c_vp, c_vp, _P(c_i64)]),
    "wrmg_plan_ns_strip": (c_i32, [_P(wrmg_mesh), c_i32, c_i32, c_i32, c_vp, c_vp, c_vp, _P(c_i64), _P(c_i32)]),
    "wrmg_loopback_create": (c_i32, [c_i32, _P(c_vp)]),
    "wrmg_loopback_destroy": (None, [c_vp]),
}
for _name, (_res, _args) in _sig.items():
    _f = getattr(lib, _name)
    _f.restype = _res
    _f.argtypes = _args


def launch_count():
    return lib.wrmg_launch_count()


def guard_violations():
    """Allocations whose guard bands were overwritten (WRMG_GUARD=1 runs)."""
    return lib.wrmg_guard_violations()


def exported_symbols():
    return sorted(_sig)


class WrmgError(RuntimeError):
    def __init__(self, status, msg, where=None):
        super().__init__(f"{STATUS.get(status, status)}: {msg}" + (f" at {where}" if where else ""))
        self.status = status
        self.where = where


def _check(st, ctx=None):
    if st != 0:
        lv, p, s = c_i32(), c_i32(), c_i32()
        msg = lib.wrmg_last_error(ctx, ctypes.byref(lv), ctypes.byref(p), ctypes.byref(s))
        where = (lv.value, p.value, s.value) if st == 4 else None
        raise WrmgError(st, (msg or b"").decode(), where)


def _ptr(t):
    """Device pointer of a float64 / int32 CUDA tensor (contiguous)."""
    import torch
    if not isinstance(t, torch.Tensor) or not t.is_cuda or not t.is_contiguous():
        raise TypeError("expected a contiguous CUDA tensor")
    return ctypes.c_void_p(t.data_ptr())


def _mesh(nx, ny, h, ncoarse, x0=0, snx=None):
    return wrmg_mesh(int(nx), int(ny), int(x0), int(nx if snx is None else snx), float(h), int(ncoarse))


STRIP_INFO = ["G0", "own0", "own1", "lg0", "nlg", "rg0", "nrg", "sl0", "nsl", "sr0", "nsr", "Lx", "Ly", "cx0", "nxl"]


def wrmg_plan_strip(gnx, gny, h, degree, rank, nranks):
    """Host-only strip plan of one rank: (info dict, global vertex ids of its patches)."""
    if gnx % nranks:
        raise ValueError("gnx must be divisible by nranks")
    snx = gnx // nranks
    m = _mesh(gnx, gny, h, 4, rank * snx, snx)
    info = np.zeros(16, dtype=np.int32)
    n = c_i64()
    _check(lib.wrmg_plan_strip(ctypes.byref(m), int(degree), int(rank), int(nranks), info.ctypes.data_as(c_vp),
                               None, ctypes.byref(n)))
    pv = np.zeros(max(n.value, 1), dtype=np.int32)
    _check(lib.wrmg_plan_strip(ctypes.byref(m), int(degree), int(rank), int(nranks), info.ctypes.data_as(c_vp),
                               pv.ctypes.data_as(c_vp), ctypes.byref(n)))
    return dict(zip(STRIP_INFO, (int(x) for x in info))), pv[:n.value]


def wrmg_plan_ns_strip(gnx, gny, h, degree, rank, nranks):
    """Host-only Navier-Stokes strip plan of one rank (lid cavity): (velocity info,
    pressure info, global vertex ids of its patches, their global sids [npatch][mp])."""
    if gnx % nranks:
        raise ValueError("gnx must be divisible by nranks")
    snx = gnx // nranks
    m = _mesh(gnx, gny, h, 4, rank * snx, snx)
    info = np.zeros(32, dtype=np.int32)
    n, mp = c_i64(), c_i32()
    _check(lib.wrmg_plan_ns_strip(ctypes.byref(m), int(degree), int(rank), int(nranks), info.ctypes.data_as(c_vp),
                                  None, None, ctypes.byref(n), ctypes.byref(mp)))
    pv = np.zeros(max(n.value, 1), dtype=np.int32)
    ps = np.zeros((max(n.value, 1), max(mp.value, 1)), dtype=np.int32)
    _check(lib.wrmg_plan_ns_strip(ctypes.byref(m), int(degree), int(rank), int(nranks), info.ctypes.data_as(c_vp),
                                  pv.ctypes.data_as(c_vp), ps.ctypes.data_as(c_vp), ctypes.byref(n),
                                  ctypes.byref(mp)))
    iu = dict(zip(STRIP_INFO, (int(x) for x in info[:16])))
    ip = dict(zip(STRIP_INFO, (int(x) for x in info[16:32])))
    return iu, ip, pv[:n.value], ps[:n.value]


def nccl_unique_id():
    """128-byte NCCL unique id (rank 0), as bytes."""
    buf = ctypes.create_string_buffer(128)
    _check(lib.wrmg_nccl_unique_id(ctypes.cast(buf, c_vp)))
    return buf.raw


class LoopbackHub:
    """In-process transport for nranks contexts driven by nranks host threads."""

    def __init__(self, nranks):
        h = c_vp()
        _check(lib.wrmg_loopback_create(int(nranks), ctypes.byref(h)))
        self.handle = h

    def close(self):
        if self.handle:
            lib.wrmg_loopback_destroy(self.handle)
            self.handle = None


def wrmg_plan(nx, ny, h, degree, q, nslabs, ncoarse=4):
    out = wrmg_layout_t()
    _check(lib.wrmg_plan(ctypes.byref(_mesh(nx, ny, h, ncoarse)), degree, q, nslabs, ctypes.byref(out)))
    return {f: getattr(out, f) for f, _ in wrmg_layout_t._fields_}


def wrmg_plan_patches(nx, ny, h, degree):
    lay = wrmg_plan(nx, ny, h, degree, 0, 1)
    npatch, mp = lay["npatch"], lay["mp_max"]
    nodes = np.empty((npatch, mp), dtype=np.int32)
    sizes = np.empty(npatch, dtype=np.int32)
    _check(lib.wrmg_plan_patches(ctypes.byref(_mesh(nx, ny, h, 4)), degree,
                                 nodes.ctypes.data_as(c_vp), sizes.ctypes.data_as(c_vp)))
    return nodes, sizes


def wrmg_batched_lu(A, piv, info, ctx=None):
    """A: (batch, m, m) float64 CUDA tensor holding column-major matrices (i.e. the
    transposes, row-major); piv (batch, m) / info (batch,) int32 CUDA tensors."""
    batch, m = A.shape[0], A.shape[1]
    st = lib.wrmg_batched_lu(ctx, _ptr(A), m, batch, _ptr(piv), _ptr(info))
    if st not in (0, 4):
        _check(st)
    return st


def wrmg_fill_uniform(out, first_id=0, seed=0, ctx=None):
    _check(lib.wrmg_fill_uniform(ctx, _ptr(out), out.numel(), int(first_id), int(seed)))


class Context:
    """One wrmg_ctx: the space-time hierarchy (heat, or Navier-Stokes with
    problem="ns": Taylor-Hood P_{degree+1}-P_degree) on one device/stream."""

    def __init__(self, nx, ny=None, h=None, degree=1, q=0, nslabs=1, dt=1.0, kappa=1.0, omega_mg=1.0,
                 nu_pre=1, nu_post=1, weights="pou", ncoarse=4, device=0, stream=None, factor_mode="auto",
                 problem="heat", reynolds=1.0, bc=None, lid_speed=1.0, rank=0, nranks=1, nccl_id=None,
                 hub=None, smoother="damped", cheb_steps=50, cheb_seed=7, scatter="atomic", orth="cgs"):
        import torch
        ny = nx if ny is None else ny
        h = 1.0 / ny if h is None else h
        if stream is None:
            stream = torch.cuda.current_stream(device).cuda_stream
        if nranks > 1:
            if nx % nranks:
                raise ValueError("strips: nx must be divisible by nranks")
            snx = nx // nranks
            self._mesh = _mesh(nx, ny, h, ncoarse, rank * snx, snx)
        else:
            self._mesh = _mesh(nx, ny, h, ncoarse)
        co = wrmg_coeffs()
        co.problem = {"heat": 0, "ns": 1}[problem]
        if bc is None:
            bc = "dirichlet0"
        co.bc = {"dirichlet0": 0, "neumann": 1, "lid": 2}[bc]
        co.kappa, co.reynolds, co.lid_speed = float(kappa), float(reynolds), float(lid_speed)
        co.weights = 0 if weights == "pou" else 1
        co.omega_mg, co.nu_pre, co.nu_post = float(omega_mg), int(nu_pre), int(nu_post)
        co.device, co.stream, co.rank, co.nranks = int(device), c_vp(stream), int(rank), int(nranks)
        self._nccl_id = None
        if nccl_id is not None:
            self._nccl_id = ctypes.create_string_buffer(bytes(nccl_id), 128)
            co.nccl_unique_id = ctypes.cast(self._nccl_id, c_vp)
        if hub is not None:
            co.loopback_hub = hub.handle
        co.smoother = {"damped": 0, "chebyshev": 1}[smoother]
        co.cheb_steps, co.cheb_seed = int(cheb_steps), int(cheb_seed)
        co.factor_mode = {"auto": 0, "lu": 1}[factor_mode]
        co.scatter = {"atomic": 0, "colour": 1}[scatter]
        co.orth = {"cgs": 0, "cgs2": 1}[orth]
        self._co = co
        h_ = c_vp()
        _check(lib.wrmg_setup(ctypes.byref(self._mesh), int(degree), int(q), int(nslabs), float(dt),
                              ctypes.byref(co), ctypes.byref(h_)))
        self._h = h_
        lay = wrmg_layout_t()
        _check(lib.wrmg_layout(self._h, ctypes.byref(lay)), self._h)
        self.layout = {f: getattr(lay, f) for f, _ in wrmg_layout_t._fields_}
        self.device = device

    # --- helpers
    def empty(self, level=None):
        import torch
        n = self.layout["ndof"] if level is None else self.level_size(level) * self.layout["nt"]
        return torch.empty(n, dtype=torch.float64, device=f"cuda:{self.device}")

    def zeros(self, level=None):
        v = self.empty(level)
        v.zero_()
        return v

    def level_size(self, level):
        n = c_i64()
        _check(lib.wrmg_level_size(self._h, int(level), ctypes.byref(n)), self._h)
        return n.value

    # --- C ABI
    def linearize(self, state=None):
        _check(lib.wrmg_linearize(self._h, None if state is None else _ptr(state)), self._h)

    def rhs(self, fhat, b):
        _check(lib.wrmg_rhs(self._h, _ptr(fhat), _ptr(b)), self._h)

    def rhs_initial(self, u0, b):
        _check(lib.wrmg_rhs_initial(self._h, _ptr(u0), _ptr(b)), self._h)

    def set_boundary_values(self, g):
        """Time-dependent Dirichlet data for Newton (NS; None restores the setup's)."""
        _check(lib.wrmg_set_boundary_values(self._h, None if g is None else _ptr(g)), self._h)

    def cheb_lambda(self, level):
        v = c_dbl()
        _check(lib.wrmg_cheb_lambda(self._h, int(level), ctypes.byref(v)), self._h)
        return v.value

    def residual(self, u, b, r, nonlinear=False):
        _check(lib.wrmg_residual(self._h, _ptr(u), _ptr(b), _ptr(r), 1 if nonlinear else 0), self._h)

    def apply(self, x, y):
        _check(lib.wrmg_apply(self._h, _ptr(x), _ptr(y)), self._h)

    def smooth(self, u, b, nsweeps=1, omega=1.0):
        _check(lib.wrmg_smooth(self._h, _ptr(u), _ptr(b), int(nsweeps), float(omega)), self._h)

    def vcycle(self, r, z):
        _check(lib.wrmg_vcycle(self._h, _ptr(r), _ptr(z)), self._h)

    def restrict(self, level, rf, rc):
        _check(lib.wrmg_restrict(self._h, int(level), _ptr(rf), _ptr(rc)), self._h)

    def prolong_add(self, level, ec, uf):
        _check(lib.wrmg_prolong_add(self._h, int(level), _ptr(ec), _ptr(uf)), self._h)

    def fgmres(self, b, x, restart=30, maxit=200, rtol=1e-8, atol=0.0):
        its, rel = c_i32(), c_dbl()
        st = lib.wrmg_fgmres(self._h, _ptr(b), _ptr(x), int(restart), int(maxit), float(rtol), float(atol),
                             ctypes.byref(its), ctypes.byref(rel))
        if st not in (0, 5, 6):
            _check(st, self._h)
        return its.value, rel.value, STATUS[st]

    def stationary(self, b, u, ncycles):
        """wrmg_stationary: ncycles of u <- u + V(b - A u) (device vectors)."""
        _check(lib.wrmg_stationary(self._h, _ptr(b), _ptr(u), int(ncycles)), self._h)

    def fgmres_host(self, bs, xs, restart=30, maxit=200, rtol=1e-8, atol=0.0):
        """wrmg_fgmres_host: solves for host (CPU, preferably pinned) float64 tensors bs[i] -> xs[i],
        uploads / downloads pipelined inside the library.  Returns (iters, relres, status)."""
        k = len(bs)
        bp = (c_vp * k)(*[b.data_ptr() for b in bs])
        xp = (c_vp * k)(*[x.data_ptr() for x in xs])
        its, rel = (c_i32 * k)(), (c_dbl * k)()
        st = lib.wrmg_fgmres_host(self._h, k, ctypes.cast(bp, c_vp), ctypes.cast(xp, c_vp), int(restart), int(maxit),
                                  float(rtol), float(atol), its, rel)
        if st not in (0, 5, 6):
            _check(st, self._h)
        return list(its), list(rel), STATUS[st]

    def newton(self, U, rtol=1e-8, maxit=20, rhs=None):
        its, lin = c_i32(), c_i32()
        st = lib.wrmg_newton_rhs(self._h, _ptr(U), None if rhs is None else _ptr(rhs), float(rtol), int(maxit),
                                 ctypes.byref(its), ctypes.byref(lin))
        if st not in (0, 6):
            _check(st, self._h)
        return its.value, lin.value, STATUS[st]

    def fill_uniform(self, out, first_id=0, seed=0):
        _check(lib.wrmg_fill_uniform(self._h, _ptr(out), out.numel(), int(first_id), int(seed)), self._h)

    def profile(self, enable=True):
        _check(lib.wrmg_profile(self._h, 1 if enable else 0), self._h)

    def kernel_stats(self):
        """{(class, level): dict(launches, ms, bytes, flops)} since profile(True)."""
        nl = self.layout["nlevels"]
        arr = (wrmg_kernel_stat * (nl * len(KERNEL_CLASSES)))()
        _check(lib.wrmg_kernel_stats(self._h, ctypes.cast(arr, c_vp)), self._h)
        out = {}
        for l in range(nl):
            for ci, name in enumerate(KERNEL_CLASSES):
                st = arr[l * len(KERNEL_CLASSES) + ci]
                if st.launches:
                    out[(name, l)] = dict(launches=st.launches, ms=st.ms, bytes=st.bytes, flops=st.flops)
        return out

    def debug_fetch(self, level, which, count, dtype=np.float64):
        out = np.empty(int(count), dtype=dtype)
        _check(lib.wrmg_debug_fetch(self._h, int(level), int(which), out.ctypes.data_as(c_vp), int(count)), self._h)
        return out

    def sync(self):
        _check(lib.wrmg_sync(self._h), self._h)

    def close(self):
        if getattr(self, "_h", None):
            lib.wrmg_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
