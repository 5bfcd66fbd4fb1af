/*
 * wrmg.h — C ABI of the B200-native waveform-relaxation multigrid hot path
 * (space-time finite elements, arXiv 2407.13997; citations are lines of the
 * paper's LaTeX source, /root/reference/PAPER.md, and readings R# of DESIGN.md).
 *
 * Discretisation: continuous Lagrange P_k (k = 1..3) in space on the structured
 * anti-diagonal triangulation of [0, nx h] x [0, ny h], upwind
 * DG(q) (q = 0..3) in time on N uniform slabs (eq. dgintime),
 * heat operator of eq. heatfem with diffusion kappa.
 *
 * Vectors.  Every vector argument is a caller-owned DEVICE pointer (e.g. a torch
 * float64 CUDA tensor's data_ptr()) holding one value per lattice node and
 * temporal DoF, waveform-major (R4):
 *     v[(i * N + n) * (q + 1) + a],   i = J * (k*nx + 1) + I,
 * i the canonical lattice node (all nodes, constrained ones included), n the
 * slab, a the temporal node.  Its length is wrmg_layout_t.ndof.  Constrained
 * (Dirichlet) DoFs are identity rows (R5).
 *
 * Streams and synchronisation.  Every call is enqueued on coeffs.stream (NULL =
 * legacy default stream) of coeffs.device and returns without synchronising,
 * except calls that return scalars to the host (wrmg_fgmres, wrmg_setup,
 * wrmg_linearize), which synchronise the stream.  Not thread-safe: one context
 * per (device, stream).
 *
 * Errors.  Every call returns a wrmg_status.  WRMG_E_SINGULAR carries the
 * (level, patch, slab) of the failing pivot (wrmg_last_error).  On error the
 * output buffers are unspecified.  Kernel-side failures are reported at the next
 * synchronising call.  No call falls back to a CPU implementation.
 *
 * Device vectors (every double * argument of the solver calls) must be 16-byte
 * aligned -- cudaMalloc and torch allocations are; a view at an odd double offset
 * is rejected with WRMG_E_INVALID (the kernels move 16-byte pairs and TMA boxes).
 */
#ifndef WRMG_H
#define WRMG_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct wrmg_ctx wrmg_ctx; /* opaque; owned by the library, freed by wrmg_destroy */

typedef enum {
  WRMG_OK = 0,
  WRMG_E_INVALID = 1,       /* bad argument (null / misaligned pointer, size, R <= 0, ...) */
  WRMG_E_UNSUPPORTED = 2,   /* degree / problem / configuration not built */
  WRMG_E_OOM = 3,           /* device allocation failed */
  WRMG_E_SINGULAR = 4,      /* |pivot| < 1e-14 * max row norm in a patch or coarse block (R10) */
  WRMG_E_BREAKDOWN = 5,     /* FGMRES: h_{j+1,j} < 1e-30 before convergence (R16) */
  WRMG_E_NOT_CONVERGED = 6, /* FGMRES: maxit reached */
  WRMG_E_CUDA = 7,          /* CUDA runtime error (message in wrmg_last_error) */
  WRMG_E_NCCL = 8
} wrmg_status;

enum { WRMG_HEAT = 0, WRMG_NAVIER_STOKES = 1 };
enum { WRMG_BC_DIRICHLET0 = 0, WRMG_BC_NEUMANN = 1, WRMG_BC_LID = 2 };
enum { WRMG_W_POU = 0, WRMG_W_NONE = 1 };  /* scatter weights W_p = 1/mu (R11) or 1 */

typedef struct {
  int32_t gnx, gny;  /* global cells per side of the anti-diagonal lattice mesh */
  int32_t x0, nx;    /* this rank's strip: first cell column and number of columns (x0 = 0, nx = gnx on 1 GPU) */
  double h;          /* cell size; domain [0, gnx h] x [0, gny h] */
  int32_t ncoarse;   /* coarsest level: coarsen while min(nx, ny) > ncoarse (R14; 0 -> 4) */
} wrmg_mesh;

typedef struct {
  int32_t problem;      /* WRMG_HEAT (WRMG_NAVIER_STOKES: WRMG_E_UNSUPPORTED in this build) */
  int32_t bc;           /* heat: WRMG_BC_DIRICHLET0 (homogeneous Dirichlet on the whole boundary) or
                           WRMG_BC_NEUMANN (homogeneous Neumann, no constrained DoF; single rank) */
  double kappa;         /* diffusion coefficient (> 0) */
  double reynolds;      /* Navier-Stokes only */
  double lid_speed;     /* Navier-Stokes only */
  int32_t weights;      /* WRMG_W_POU (default) | WRMG_W_NONE */
  double omega_mg;      /* smoother damping inside the V-cycle (R15; 0 -> 1.0) */
  int32_t nu_pre, nu_post; /* V(nu_pre, nu_post) (R15; 0,0 -> 1,1) */
  int32_t factor_mode;  /* 0 AUTO: heat patch solves Kronecker-diagonalised (kernels_kron.cu), N <= 256;
                           1 LU: per-class LU factors (H5) applied by the split-form sweep */
  int32_t device;       /* CUDA device ordinal */
  void *stream;         /* cudaStream_t; NULL = default stream */
  int32_t rank, nranks; /* strip partition across ranks (heat): rank r of nranks
                           owns cell columns [mesh.x0, mesh.x0 + mesh.nx) with x0 = r * nx, nx * nranks = gnx */
  const void *nccl_unique_id; /* nranks > 1: 128-byte ncclUniqueId from wrmg_nccl_unique_id on rank 0 */
  void *loopback_hub;   /* nranks > 1 without NCCL: hub of wrmg_loopback_create, ranks = host threads of one
                           process sharing one device (tests); NULL = NCCL */
  int32_t smoother;     /* WRMG_SMOOTH_DAMPED (default: nu damped additive sweeps, R15) |
                           WRMG_SMOOTH_CHEBYSHEV (nu Chebyshev-accelerated steps on [0.25 lam, 1.05 lam], lam from
                           cheb_steps Arnoldi steps on B A per level -- re-estimated by every Navier-Stokes
                           linearisation, DESIGN.md R-cheb; single rank) */
  int32_t cheb_steps;   /* Arnoldi steps of the lambda estimate (0 -> 50, <= 63) */
  uint64_t cheb_seed;   /* seed of the Arnoldi start vector (R6 generator at canonical ids) */
  int32_t scatter;      /* weighted additive scatter (H8) of the heat sweep in factor_mode AUTO:
                           WRMG_SCATTER_ATOMIC (default; FP64 atomics, order of the <= mu_max additions per
                           value unspecified) | WRMG_SCATTER_COLOUR (three passes, one per vertex colour
                           (i - j) mod 3 -- patches of one colour share no DoF -- so every value receives one
                           addition per pass in a fixed order: bitwise reproducible) */
  int32_t orth;         /* Arnoldi orthogonalisation of wrmg_fgmres (R16): WRMG_ORTH_CGS (default;
                           classical Gram-Schmidt, one pass -- the default of the PETSc FGMRES that the
                           paper's Firedrake runs use) | WRMG_ORTH_CGS2 (applied twice) */
} wrmg_coeffs;
enum { WRMG_SMOOTH_DAMPED = 0, WRMG_SMOOTH_CHEBYSHEV = 1 };
enum { WRMG_SCATTER_ATOMIC = 0, WRMG_SCATTER_COLOUR = 1 };
enum { WRMG_ORTH_CGS = 0, WRMG_ORTH_CGS2 = 1 };

typedef struct {
  int64_t nnode;        /* lattice nodes of the finest level owned by this rank */
  int64_t nt;           /* temporal DoFs per node, N (q + 1) */
  int64_t ndof;         /* vector length nnode * nt */
  int64_t nfree_st;     /* free (unconstrained) space-time DoFs */
  int32_t lx, ly;       /* lattice nodes per direction: k nx + 1, k ny + 1 */
  int32_t nlevels;      /* multigrid levels (coarse + ... + fine) */
  int32_t degree, q, nslabs;
  int64_t npatch;       /* finest-level patches (R8) */
  int32_t mp_max;       /* largest spatial patch size */
  int32_t npatch_types; /* distinct finest-level patch blocks factored (translation classes) */
  int64_t smooth_dof_updates_per_vcycle; /* sum over levels >= 1 of free space-time DoFs x (nu_pre + nu_post)
                                            (owned DoFs on a strip) */
  int32_t own0, own1;   /* owned lattice columns [own0, own1] of the local lattice (0, lx-1 on one rank) */
  int32_t g0;           /* global lattice column of local column 0 */
  int64_t nfree_owned_st; /* free space-time DoFs owned by this rank */
  /* Navier-Stokes (lx, ly, own0, own1, g0 above describe the velocity lattice; sids
     u_x: [0, lu), u_y: [lu, 2 lu), p: [2 lu, 2 lu + lpx lpy)); 0 for the heat operator */
  int64_t lu;             /* velocity lattice nodes lx * ly */
  int32_t lpx, lpy;       /* pressure lattice nodes per direction */
  int32_t own0p, own1p;   /* owned pressure lattice columns */
  int32_t g0p;            /* global pressure lattice column of local column 0 */
} wrmg_layout_t;

/* Build the hierarchy on the device.  PAPER.md:351-360 (space-only coarsening),
 * PAPER.md:381 (P = I (x) P_h, vertex-star patches).  Host: lattice maps, CSR
 * patterns and patch tables (integer setup, H3).  Device kernels: spatial
 * assembly (H1), patch blocks (H4), batched LU (H5), coarse factorisation.
 * degree = k in {1,2,3}; q in {0,1,2,3}; nslabs = N >= 1; dt > 0.
 * Synchronises.  *out receives the context (NULL on error). */
wrmg_status wrmg_setup(const wrmg_mesh *mesh, int32_t degree, int32_t q, int32_t nslabs, double dt,
                       const wrmg_coeffs *coeffs, wrmg_ctx **out);

/* Sizes of the finest level (host struct filled). */
wrmg_status wrmg_layout(const wrmg_ctx *ctx, wrmg_layout_t *out);

/* (Re)factorise every patch and coarse block for the operator linearised at
 * `state` (device vector, NULL for the linear heat operator).  Heat: recomputes
 * H1/H4/H5 on the device.  Synchronises; WRMG_E_SINGULAR on a failed pivot.
 * Navier-Stokes: the Vanka inverses (m^2 doubles per (patch, slab)) of a level
 * whose store does not fit the device (92 % of the free memory at setup less
 * 8 GB) are kept for a window of W slabs only: this call factors every
 * window once for the singularity check, and every sweep of that level
 * re-factors each window before sweeping it (PAPER.md:390 fixes the patch solve,
 * not its storage; DESIGN.md 1b "slab windows").  Environment: WRMG_NS_WINDOW=W
 * forces W-slab windows, WRMG_NS_STORE_GB sets the budget. */
wrmg_status wrmg_linearize(wrmg_ctx *ctx, const double *state);

/* b = (M (x) I_N (x) Mt) fhat on free rows, bc value on constrained rows
 * (forcing term of eq. heatfem with f = sum fhat phi; R6).  fhat: ndof values. */
wrmg_status wrmg_rhs(wrmg_ctx *ctx, const double *fhat, double *b);

/* b += the initial-state term of eq. dgintime (Y_0^- = y_0, R7): on every free row
 * i and temporal node a of slab 0, phi_a(0) (M u0)_i, M the spatial mass (heat) or
 * the velocity mass M2 (Navier-Stokes; the jump acts on velocity only).  u0:
 * nnode (heat) / sid (NS) nodal values on the device. */
wrmg_status wrmg_rhs_initial(wrmg_ctx *ctx, const double *u0, double *b);

/* Navier-Stokes: time-dependent Dirichlet data (R5, R28).  g: device or
 * host vector of ndof values in the solution layout; only its constrained rows
 * (boundary velocity DoFs, every slab and temporal node) are read, and
 * wrmg_newton / wrmg_newton_rhs then impose U = g there instead of the setup's
 * per-sid values (bc, lid_speed).  Copied (the caller keeps ownership);
 * g = NULL restores the setup's values.  Synchronises.  Heat contexts:
 * WRMG_E_UNSUPPORTED.  Used for the Chorin problem, whose
 * exact velocity decays in time on the boundary. */
wrmg_status wrmg_set_boundary_values(wrmg_ctx *ctx, const double *g);

/* Largest-eigenvalue estimates of the Chebyshev smoother (R-cheb), level >= 1
 * (0 for the coarsest / damped smoothing).  Host output. */
wrmg_status wrmg_cheb_lambda(const wrmg_ctx *ctx, int32_t level, double *lam);

/* r = b - A u on the finest level (H6; eq. heatfem; constrained rows r = b - u).
 * `nonlinear` (Navier-Stokes): r = b - F(u).  r may not alias u or b.
 * Strips (nranks > 1): rows of owned columns are valid; the ghost columns of u
 * are refreshed from the neighbours first (u is written there). */
wrmg_status wrmg_residual(wrmg_ctx *ctx, const double *u, const double *b, double *r, int32_t nonlinear);

/* y = A x (Krylov matvec; constrained rows y = x). */
wrmg_status wrmg_apply(wrmg_ctx *ctx, const double *x, double *y);

/* nsweeps additive waveform-relaxation sweeps on the finest level, in place on u
 * (H6 + H7 + H8, R9-R11):
 *   r = b - A u;  for every patch p, for n = 0..N-1:  x_{p,n} = D_p^{-1}(r_{p,n} - L_p x_{p,n-1});
 *   u += omega * sum_p R_p^T W_p x_p. */
wrmg_status wrmg_smooth(wrmg_ctx *ctx, double *u, const double *b, int32_t nsweeps, double omega);

/* z = B r: one V(nu_pre, nu_post) cycle from a zero initial guess (H9-H12;
 * PAPER.md:361-366).  r must vanish on constrained rows (corrections, R5).
 * Strips: r is read on owned columns (its ghost columns are overwritten); z is
 * valid on owned and ghost columns; the coarsest level is solved replicated
 * after an all-gather. */
wrmg_status wrmg_vcycle(wrmg_ctx *ctx, const double *r, double *z);

/* Restriction / prolongation between finest-level `level` (>= 1, counted from the
 * coarsest = 0) and level-1 (H9, H10; PAPER.md:381 R = P^T, P = I (x) P_h).  The
 * vectors have the layouts of the respective levels (wrmg_level_size). */
wrmg_status wrmg_restrict(wrmg_ctx *ctx, int32_t level, const double *r_fine, double *r_coarse);
wrmg_status wrmg_prolong_add(wrmg_ctx *ctx, int32_t level, const double *e_coarse, double *u_fine);
/* Number of lattice nodes of a level (vector length = nodes * nt). */
wrmg_status wrmg_level_size(const wrmg_ctx *ctx, int32_t level, int64_t *nnode);

/* Right-preconditioned FGMRES(restart) with CGS2, x0 = 0 (H13; PAPER.md:361-366,
 * R16).  Stops when |g_{j+1}| <= max(rtol ||b||, atol).  x receives the iterate,
 * *iters the number of preconditioner applications, *relres the final true
 * relative residual ||b - A x|| / ||b||.  Synchronises every Arnoldi step.
 * Strips (nranks > 1): collective - every rank calls it with its local b and x;
 * b is read on owned columns, x is valid on owned and ghost columns; dot products
 * run over owned rows and are summed across ranks (all-gather of the per-rank
 * partial results, added in rank order, so every rank takes identical decisions).
 * Returns WRMG_OK, WRMG_E_BREAKDOWN or WRMG_E_NOT_CONVERGED (x still valid). */
wrmg_status wrmg_fgmres(wrmg_ctx *ctx, const double *b, double *x, int32_t restart, int32_t maxit,
                        double rtol, double atol, int32_t *iters, double *relres);

/* ncycles stationary multigrid iterations u <- u + B (b - A u), B = one wrmg_vcycle (the C5
 * protocol: 20 V(1,1) cycles from u = 0).  u, b: device vectors as for
 * wrmg_residual (strips: u's ghost columns are refreshed).  Two scratch vectors are owned by
 * the context (allocated at the first call). */
wrmg_status wrmg_stationary(wrmg_ctx *ctx, const double *b, double *u, int32_t ncycles);

/* Serving form of wrmg_fgmres on HOST buffers: solves A x_i = b_i for nrhs right-hand sides
 * b_host[i] -> x_host[i] (each ndof doubles in the owned layout of wrmg_layout; page-locked
 * memory recommended, pageable accepted).  The library owns two device input and two output
 * buffers and a copy stream: the upload of b_{i+1} and the download of x_{i-1} run on the copy
 * engines while right-hand side i is solved.  iters / relres (may be NULL) receive nrhs
 * values.  Returns the first non-OK status of the solves (all are attempted); the host
 * results are complete when the call returns. */
wrmg_status wrmg_fgmres_host(wrmg_ctx *ctx, int32_t nrhs, const double *const *b_host, double *const *x_host,
                             int32_t restart, int32_t maxit, double rtol, double atol, int32_t *iters,
                             double *relres);

/* Navier-Stokes Newton-FGMRES-WRMG (H14, R22): solves F(U) = 0
 * from U (constrained rows set to the boundary values), relinearising every
 * level and refactorising every (patch, slab) block at each step, FGMRES(30)
 * with Eisenstat-Walker forcing (eta_0 = 0.3), until ||F|| <= rtol ||F(U_0)||.
 * *newton_its = linear solves, *lin_its = total FGMRES iterations.
 * WRMG_E_NOT_CONVERGED after maxit steps (U holds the last iterate). */
wrmg_status wrmg_newton(wrmg_ctx *ctx, double *U, double rtol, int32_t maxit, int32_t *newton_its,
                        int32_t *lin_its);
/* As wrmg_newton for F(U) = rhs (rhs on free rows, NULL = 0): e.g. the
 * initial-state term of wrmg_rhs_initial for one slab of a timestepping run. */
wrmg_status wrmg_newton_rhs(wrmg_ctx *ctx, double *U, const double *rhs, double rtol, int32_t maxit,
                            int32_t *newton_its, int32_t *lin_its);

/* Batched dense LU with partial pivoting (H5, R10) on caller device memory:
 * A holds `batch` column-major m x m matrices (A + b*m*m), overwritten by the
 * factors (unit-lower L below the diagonal, U on and above, LAPACK dgetrf
 * layout); piv (batch*m int32) receives 0-based pivot rows; info (batch int32)
 * receives 0 or 1 + the first singular column.  Synchronises.
 * Returns WRMG_E_SINGULAR if any info != 0. */
wrmg_status wrmg_batched_lu(const wrmg_ctx *ctx, double *A, int32_t m, int32_t batch, int32_t *piv,
                            int32_t *info);

/* Counter-based generator of R6 (splitmix64 finaliser) on the device:
 * out[t] = U[-1,1) at canonical id first_id + t, t < count. */
wrmg_status wrmg_fill_uniform(const wrmg_ctx *ctx, double *out, int64_t count, uint64_t first_id,
                              uint64_t seed);

/* Wait for all work enqueued on the context's stream; reports deferred kernel errors. */
wrmg_status wrmg_sync(wrmg_ctx *ctx);

/* Last error message (thread-local when ctx is NULL); level/patch/slab of a
 * singular pivot when the last status was WRMG_E_SINGULAR (else -1). */
const char *wrmg_last_error(const wrmg_ctx *ctx, int32_t *level, int32_t *patch, int32_t *slab);

/* Free every device and host resource of the context. */
void wrmg_destroy(wrmg_ctx *ctx);

/* Kernel timing.  wrmg_profile(ctx, 1) resets the counters and, until
 * wrmg_profile(ctx, 0), records a CUDA event pair on the context's stream around
 * every hot-path launch (classes below).  wrmg_kernel_stats synchronises and
 * fills out[level * WRMG_K_COUNT + cls] for levels 0..nlevels-1 (level 0 =
 * coarsest): launch count, summed device milliseconds, and the algorithmic
 * bytes / flops of those launches ("Roofline accounting"). */
enum { WRMG_K_RESIDUAL = 0, WRMG_K_SWEEP = 1, WRMG_K_RESTRICT = 2, WRMG_K_PROLONG = 3, WRMG_K_COARSE = 4,
       WRMG_K_KRYLOV = 5, WRMG_K_FACTOR = 6, WRMG_K_COUNT = 7 };
typedef struct {
  int64_t launches;
  double ms;
  double bytes;
  double flops;
} wrmg_kernel_stat;
wrmg_status wrmg_profile(wrmg_ctx *ctx, int32_t enable);
wrmg_status wrmg_kernel_stats(wrmg_ctx *ctx, wrmg_kernel_stat *out);

/* Test / introspection hook: copy `count` elements of an internal device array of
 * `level` to host memory.  which: 0 spatial val (heat M, NS M2), 1 val2 (heat
 * kappa K, NS K2 + divergence blocks), 2 NS convection [nvv][N(q+1)], 3 NS
 * injected state, 4 NS coarse slab blocks after factorisation (LU, column-major,
 * per slab), 5 CSR rowptr (int32), 6 CSR col (int32), 7 coarse free sids (int32),
 * 8 NS coarse LU info per slab (int32), 9 NS coarse LU pivots (int32).
 * Synchronises.  WRMG_E_INVALID if the array is absent or shorter than count. */
wrmg_status wrmg_debug_fetch(wrmg_ctx *ctx, int32_t level, int32_t which, void *host_dst, int64_t count);

/* Strip partition transports.  wrmg_nccl_unique_id writes a 128-byte NCCL unique
 * id (call on rank 0, broadcast, pass as coeffs.nccl_unique_id on every rank).
 * wrmg_loopback_create makes an in-process hub for nranks contexts driven by
 * nranks host threads on one device (halo hand-over by host barrier + device
 * copies); destroy it after every context using it. */
wrmg_status wrmg_nccl_unique_id(void *out128);
wrmg_status wrmg_loopback_create(int32_t nranks, void **hub);
void wrmg_loopback_destroy(void *hub);

/* Number of kernels this library has launched in the process so far. */
int64_t wrmg_launch_count(void);
/* Host-only: allocations whose guard bands were found overwritten when they were freed.
 * Guard bands (4 KB of 0xFF on both sides of every device allocation of the library) are
 * enabled by the environment variable WRMG_GUARD=1 at the first allocation; 0 otherwise. */
int64_t wrmg_guard_violations(void);

/* Host-only planning query (no device needed): sizes of the finest level and
 * hierarchy for a configuration, for tests of the host setup logic (H3). */
wrmg_status wrmg_plan(const wrmg_mesh *mesh, int32_t degree, int32_t q, int32_t nslabs,
                      wrmg_layout_t *out);

/* Host-only: the finest-level patch table (H3, R8).  nodes receives npatch *
 * mp_max int32 canonical node ids (-1 padded), sizes npatch int32 sizes; either
 * may be NULL.  Buffers are host memory owned by the caller. */
wrmg_status wrmg_plan_patches(const wrmg_mesh *mesh, int32_t degree, int32_t *nodes, int32_t *sizes);

/* Host-only test hook: eigenvalues (wr + i wi) of the n x n row-major upper
 * Hessenberg H by the Francis double-shift QR iteration used for the Chebyshev
 * eigenvalue estimate (R-cheb).  WRMG_E_NOT_CONVERGED if the iteration fails. */
wrmg_status wrmg_hessenberg_eig(const double *H, int32_t n, double *wr, double *wi);

/* Host-only: the strip plan of one rank (mesh->x0, mesh->nx
 * its cell columns).  info[16] = {G0, own0, own1, lg0, nlg, rg0, nrg, sl0, nsl,
 * sr0, nsr, Lx, Ly, cx0, nxl, 0}: global column of local column 0, owned local
 * columns, left / right ghost columns, columns sent left / right, local lattice
 * size, local cells.  patch_vertex (may be NULL) receives the global vertex id
 * J (gnx + 1) + I of each owned patch, *npatch their count. */
wrmg_status wrmg_plan_strip(const wrmg_mesh *mesh, int32_t degree, int32_t rank, int32_t nranks, int32_t *info,
                            int32_t *patch_vertex, int64_t *npatch);

/* Host-only: the Navier-Stokes strip plan of one rank (Taylor-Hood P_{degree+1} -
 * P_degree; the lid-cavity boundary).  info[32] = the 16
 * entries of wrmg_plan_strip for the velocity lattice, then for the pressure
 * lattice.  *npatch, *mp: owned Vanka+star patches and the largest size; when
 * patch_vertex / patch_sids are not NULL they receive each patch's global vertex
 * id and its sids as GLOBAL sids ([npatch][mp], -1 padded). */
wrmg_status wrmg_plan_ns_strip(const wrmg_mesh *mesh, int32_t degree, int32_t rank, int32_t nranks, int32_t *info,
                               int32_t *patch_vertex, int32_t *patch_sids, int64_t *npatch, int32_t *mp);

#ifdef __cplusplus
}
#endif
#endif /* WRMG_H */
