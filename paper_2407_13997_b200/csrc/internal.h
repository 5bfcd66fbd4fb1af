// Internal declarations of libwrmg (not part of the C ABI).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <cstdio>
#include <string>
#include <vector>

#include "../../include/wrmg.h"

namespace wrmg {

constexpr int kMaxQ = 3;            // DG(q), q <= 3
constexpr int kMaxK = 3;            // CG(k), k <= 3
constexpr int kMaxLoc = 10;         // (k+1)(k+2)/2 for k = 3

// ---------------------------------------------------------------- host math
// Reference P_k element on T^ = {xi, eta >= 0, xi + eta <= 1} with nodes
// (a/k, b/k); local index ordering: b outer, a inner (see host_fem.cu).
struct RefElement {
  int k = 0, nloc = 0;
  int a[kMaxLoc], b[kMaxLoc];
  double M[kMaxLoc * kMaxLoc];   // int phi_i phi_j over T^
  double K[kMaxLoc * kMaxLoc];   // int grad phi_i . grad phi_j over T^
};
void build_ref_element(int k, RefElement *out);
// Values of the reference basis at the point with k*lambda = (kl0, kl1, kl2)
// (barycentric coordinates times k; exact rationals keep lattice zeros exact).
void eval_basis_klambda(int k, double kl1, double kl2, double *vals);

struct Temporal {
  int q = 0, nq = 1;
  double CE[(kMaxQ + 1) * (kMaxQ + 1)];  // C + E0, row a, column b
  double Mt[(kMaxQ + 1) * (kMaxQ + 1)];  // dt int phi_a phi_b
  double E1[(kMaxQ + 1) * (kMaxQ + 1)];  // phi_a(0) phi_b(1)
  double T[(kMaxQ + 1) * (kMaxQ + 1) * (kMaxQ + 1)];  // dt int phi_a phi_b phi_c, index (a nq + b) nq + c
  double phi0[kMaxQ + 1];                             // phi_a(0)
};
void build_temporal(int q, double dt, Temporal *out);
// Reference basis of degree k (local order of lattice.h) and its xi/eta derivatives at (xi, eta).
void eval_basis_grad(int k, double xi, double eta, double *v, double *dxi, double *deta);
// Collapsed (Duffy) Gauss rule with ng x ng points on the reference triangle.
void gauss_triangle(int ng, std::vector<double> &xi, std::vector<double> &eta, std::vector<double> &w);

// Residual stencil classes (kernels_residual.cu), passed by value as a kernel parameter.
constexpr int kStencilMaxC = 16, kStencilMaxE = 40;
struct StencilTab {
  int ncls;
  int cnt[kStencilMaxC];
  int32_t off[kStencilMaxC][kStencilMaxE];   // (dJ * RW + dI) * 32 (q+1): smem offset (8x8 tiles, 32 slabs)
  double m[kStencilMaxC][kStencilMaxE], kk[kStencilMaxC][kStencilMaxE];
};

// Macro-block residual (kernels_residual_mac.cu): interior coefficients of every
// row type (I mod k, J mod k) in the entry order of residual_mac_gen.h, and the
// stencil class that holds them.
constexpr int kMacMaxEntries = 153;  // P3: 9 row types, 153 stencil entries
struct MacCoef {
  double m[kMacMaxEntries], k[kMacMaxEntries];
};
struct MacTab {
  MacCoef C;
  int32_t canon[9];
};

// Symmetry-reduced patch solve of the interior vertex-star class (host_sym.cu,
// kernels_sweep_sym.cu): character blocks V_chi, per-mode DG(q) inverses.
constexpr int kSymMaxMP = 19;
struct SymTab {
  double V[7 * 7 + 3 * 3 + 4 * 4 + 5 * 5];
  double S[kSymMaxMP * 16];
  double sig[kSymMaxMP];
  double sig2[5][kSymMaxMP];  // sig^(2^k), the shuffle-scan coefficients (host_sym.cu)
};

// 2 x 2 vertex tiles of the symmetric class (kernels_sweep_sym.cu, tiled form): the
// union of the four patches' nodes (relative lattice offsets from the tile's first
// vertex node), which of them no patch outside the tile touches (plain
// read-modify-write instead of atomics), and the (patch, slot) pairs feeding each.
constexpr int kTileMaxU = 64;
struct TileGeom {
  int nu = 0;
  int32_t off[kTileMaxU];
  uint8_t interior[kTileMaxU];
  uint8_t cnt[kTileMaxU];
  int16_t src[kTileMaxU][4];  // w * MP + slot
};

// Work lists of one sweep pass (coloured scatter: one per vertex colour (i - j) mod 3,
// whose patches share no node, so each value receives one addition per pass and the
// sweep is bitwise deterministic).
struct SweepLists {
  int ncta = 0, pp = 1;
  int32_t *cta_patch = nullptr, *cta_type = nullptr;   // k_sweep_kron
  int ngrp8 = 0;
  int32_t *grp_patch8 = nullptr, *grp_type8 = nullptr; // k_sweep_kron_mma
  int64_t nsym = 0;
  int32_t *sym_list = nullptr;                          // k_sweep_sym (indices into sym_nodes)
};

// Spatial strip of a level on this rank (host_strip.cu).
struct StripInfo {
  int rank = 0, nranks = 1;
  int gnx = 0, x0 = 0, nx = 0;  // global cells, this rank's cell columns
  int cx0 = 0, nxl = 0;         // local mesh: cells [cx0, cx0 + nxl)
  int G0 = 0;                   // global node column of local column 0 (= k cx0)
  int own0 = 0, own1 = 0;       // owned local columns [own0, own1] (inclusive)
  int lg0 = 0, nlg = 0;         // left ghost local columns [lg0, lg0 + nlg)
  int rg0 = 0, nrg = 0;         // right ghost local columns
  int sl0 = 0, nsl = 0;         // columns sent to the left rank (its right ghosts)
  int sr0 = 0, nsr = 0;         // columns sent to the right rank (its left ghosts)
};
struct Comm;

// ---------------------------------------------------------------- device data
struct DevCSR {
  int64_t nrow = 0, nnz = 0;
  int32_t *rowptr = nullptr, *col = nullptr;
  double *val = nullptr, *val2 = nullptr;  // M and K (spatial) or P entries
};

struct Level {
  int nx = 0, ny = 0;
  double h = 0;
  int Lx = 0, Ly = 0;
  int64_t nnode = 0, nfree = 0;
  DevCSR A;                         // spatial M (val) and kappa K (val2), all nodes
  uint8_t *con = nullptr;           // constrained mask
  std::vector<uint8_t> h_con;
  // patches (vertex-star, R8)
  int64_t npatch = 0;
  int mp = 0;                       // padded spatial patch size (compile-time class)
  int ntypes = 0;
  int32_t *pnodes = nullptr;        // [npatch][mp], -1 pad
  int32_t *ptype = nullptr;         // [npatch]
  double *wnode = nullptr;          // 1/mu_i (or 1) per node, 0 on nodes in no patch
  int32_t *type_rep = nullptr;      // representative patch of each type
  double *Dblk = nullptr;           // [ntypes][m][m] assembled local blocks (column-major), m = nq*mp
  double *Dinv = nullptr;           // [ntypes][m][m] row-major inverses
  double *G = nullptr;              // [ntypes][m][mp] jump propagator Dinv[:, a=0] M_p
  int32_t *piv = nullptr, *info = nullptr;
  std::vector<int32_t> h_type_rep;
  // Kronecker-diagonalised sweep (kernels_kron.cu): per class V (mp x ld), V^T, S, sigma
  double *kV = nullptr, *kVT = nullptr, *kS = nullptr, *ksig = nullptr;
  int32_t *cta_patch = nullptr, *cta_type = nullptr;
  int kron_pp = 1, kron_ncta = 0;
  int32_t *cta_patch1 = nullptr, *cta_type1 = nullptr;  // one patch per CTA (DMMA sweep)
  int kron_ncta1 = 0;
  int32_t *grp_patch8 = nullptr, *grp_type8 = nullptr;  // class-pure groups of 8 patches (DMMA sweep)
  int kron_ngrp8 = 0;
  // residual stencil classes
  uint8_t *rcls = nullptr;
  std::vector<int32_t> h_cls_rep;
  bool stencil_ok = false;
  StencilTab stencil{};
  int64_t *goff = nullptr;  // [kStencilMaxC][kStencilMaxE] global element offsets (dJ Lx + dI) NT
  std::vector<uint8_t> h_rcls;      // host copy of rcls
  bool mac_ok = false;              // macro-block residual available on this level
  MacTab mac{};
  int32_t *gen_rows = nullptr;      // rows outside the interior classes (fix-up after the macro kernel)
  int64_t ngen_rows = 0;
  // symmetry-reduced sweep of the interior patch class (the kron work lists then hold the other classes)
  bool sym_ok = false;
  int sym_cls = -1;
  int64_t nsym = 0;
  int32_t *sym_nodes = nullptr;     // [nsym][mp] patch nodes in host_sym.cu slot order
  std::vector<int64_t> sym_pos;     // [mp][mp] CSR positions of the representative's block (-1: none)
  SymTab symtab{};
  int64_t ntile = 0, nsingle = 0;
  int32_t *tile_patch = nullptr;    // [ntile][4] indices into sym_nodes (tile vertices (0,0),(1,0),(0,1),(1,1))
  int32_t *sym_single = nullptr;    // sym patches outside complete tiles
  TileGeom tgeo{};
  TileGeom *tgeo_dev = nullptr;
  bool coloured = false;            // WRMG_SCATTER_COLOUR: per-colour work lists below
  SweepLists col[3];
  // transfer from this level to the next finer (stored on the coarse side)
  DevCSR P;    // rows: fine nodes, cols: coarse nodes
  DevCSR R;    // rows: coarse nodes, cols: fine nodes (R = P^T, same doubles)
  // V-cycle work vectors (levels below the finest)
  double *vr = nullptr, *vz = nullptr, *vt = nullptr;
  // Navier-Stokes (Taylor-Hood) level: A = sid CSR with val = M2, val2 = K2 + divergence blocks
  int64_t Lu = 0, Lp = 0;
  int Lux = 0, Lpx = 0;
  int32_t *vvptr = nullptr;         // [2 Lu + 1] compact index of velocity-velocity entries
  int64_t nvv = 0;
  double *conv = nullptr;           // [nvv][NT]: R N(w_{n,c}) of the current linearisation
  double *state = nullptr;          // injected linearisation state (levels below the finest)
  int64_t mstride = 0;              // doubles per stored (patch, slab) inverse
  double *nsinv = nullptr;          // [npatch][nswin][mstride] column-major D_{p,n}^{-1}
  int nswin = 0;                    // stored slabs per patch: N, or a window recomputed in every sweep
  double *nsxs = nullptr;           // windows: [npatch][m] patch solution at the end of the previous window
  int32_t *nsinfo = nullptr;        // [npatch][N]
  int32_t *ppos = nullptr, *pvv = nullptr;  // [npatch][mp][mp] CSR / convection index of each patch pair
  int64_t nsfree_patch_dofs = 0;    // sum of patch sizes (algorithmic accounting)
  // strip partition (nranks > 1)
  StripInfo st;                     // heat: the lattice; Navier-Stokes: the velocity lattice
  StripInfo stp;                    // Navier-Stokes: the pressure lattice
  int64_t gLp = 0;                  // Navier-Stokes: global pressure nodes (strip projection)
  double *hx[4] = {nullptr, nullptr, nullptr, nullptr};  // halo send-left, recv-left, send-right, recv-right
  int64_t nfree_owned = 0;
};

struct Coarse {
  int64_t nfree = 0;
  int m = 0, mp = 0;
  int32_t *nodes = nullptr;   // free coarse nodes (canonical order)
  double *Dblk = nullptr;     // m x m, column-major
  double *DinvT = nullptr;    // m x m, column-major inverse (Dinv^T row-major)
  double *Gq = nullptr;       // mp x mp row-major: end-trace propagator
  double *GT = nullptr;       // mp x m: G transposed (G[rho][j] at GT[j*m + rho])
  double *kV = nullptr, *kVT = nullptr, *kS = nullptr, *ksig = nullptr;  // Kronecker coarse solve
  double *Z = nullptr;        // N x m scratch
  double *Y = nullptr;        // (N+1) x mp scratch
  int32_t *piv = nullptr, *info = nullptr;
  // Navier-Stokes coarse solve: per-slab blocks with the pinned pressure DoF (R19)
  int pin = -1;
  int nnzj = 0;               // CSR entries of the free coarse rows (jump mass rows staged by the solve)
  double *nsD = nullptr, *nsinvT = nullptr, *xq = nullptr;
  int32_t *nspiv = nullptr, *nsinfo = nullptr;
  // parallel-in-time form of the NS coarse march (only the velocity end trace
  // propagates): H_n = D_n^{-1} E (m x mp per slab, column-major), G_n = its a = q
  // rows (mp x mp, column-major), scratch z_n = D_n^{-1} r_n (N x m), y_n (N x mp)
  double *nsH = nullptr, *nsG = nullptr, *nsZ = nullptr, *nsY = nullptr;
  int32_t *sid2c = nullptr;   // sid -> coarse free index or -1
};

}  // namespace wrmg

struct wrmg_ctx {
  wrmg_mesh mesh{};
  wrmg_coeffs co{};
  int k = 1, q = 0, N = 1, nq = 1;
  int64_t nt = 1;
  double dt = 0;
  cudaStream_t stream = nullptr;
  // side stream + events: the boundary-class sweep kernels run concurrently with the
  // symmetric-class one (both add into u with FP64 atomics)
  cudaStream_t side = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  wrmg::RefElement ref;
  wrmg::Temporal tm;
  std::vector<wrmg::Level> lv;  // 0 = coarsest
  wrmg::Coarse coarse;
  double *ref_dev = nullptr;    // reference M^, K^ on device
  // FGMRES work space
  int restart_alloc = 0;
  std::vector<double *> V, Z;
  double *w = nullptr, *red = nullptr, *red_host = nullptr;
  double *kry = nullptr;   // device-side CGS2 coefficients of the single-rank FGMRES (kernels_krylov.cu)
  // wrmg_fgmres_host: double-buffered device copies of b / x, copy stream, events
  double *hb[2] = {nullptr, nullptr}, *hx[2] = {nullptr, nullptr};
  double *st_r = nullptr, *st_z = nullptr;  // wrmg_stationary scratch
  cudaStream_t copy = nullptr;
  cudaEvent_t ev_in[2] = {nullptr, nullptr}, ev_solved[2] = {nullptr, nullptr}, ev_out[2] = {nullptr, nullptr};
  double *hmap = nullptr;  // mapped pinned host buffer (2 x hmap_cap doubles): small Krylov results without the copy engines
  int hmap_cap = 0;        // doubles per direction: max(1024, 64 nranks)
  double *gred = nullptr;  // strips: all ranks' reduction results (nranks x 64), for wrmg_fgmres
  double *tmp = nullptr;        // finest-level scratch (residual)
  bool use_kron = true;         // factor_mode AUTO: Kronecker-diagonalised heat patch solves
  bool coarse_kron = false;     // the coarsest level's solve in Kronecker form (mp <= kCoarseKronMax)
  std::string err;
  int err_level = -1, err_patch = -1, err_slab = -1;
  // kernel timing (wrmg_profile / wrmg_kernel_stats)
  struct ProfRec {
    int cls, lvl;
    cudaEvent_t a, b;
    double bytes, flops;
  };
  bool prof_on = false;
  std::vector<ProfRec> prof_recs;
  std::vector<cudaEvent_t> prof_pool;
  wrmg_kernel_stat stats[WRMG_K_COUNT][16];
  std::vector<double> sweep_flops;  // per level: algorithmic flops of one sweep
  // Navier-Stokes
  bool ns = false;
  double *th_ref = nullptr, *th_T = nullptr;   // Taylor-Hood reference integrals on the device
  int th_nu = 0, th_np = 0;
  double *bcg = nullptr;                       // finest-level boundary values per sid
  double *bcg_st = nullptr;                    // wrmg_set_boundary_values: per space-time DoF (NULL: bcg)
  double *proj = nullptr;                      // pressure-projection scratch
  double *conv_nl = nullptr;                   // finest R O(U) for the nonlinear residual
  double *nl_b = nullptr, *nl_r = nullptr, *nl_dx = nullptr;  // Newton work vectors
  // strip partition (nranks > 1): transport, replicated global coarsest level
  bool strip = false;
  wrmg::Comm *comm = nullptr;
  wrmg::Level gco;
  // strips whose coarse levels are narrower than 2 cells per rank: those levels run
  // replicated as a single-rank hierarchy; xfer holds P / R between the coarsest
  // partitioned level (owned rows) and the replicated finest level (global ids)
  wrmg_ctx *sub = nullptr;
  wrmg::Level xfer;
  double *sub_r = nullptr, *sub_z = nullptr, *sub_part = nullptr, *sub_all = nullptr;
  double *gr = nullptr, *gz = nullptr, *gsend = nullptr, *grecv = nullptr;
  int64_t gchunk = 0;
  // Navier-Stokes strips: state refresh (all-gather of the owned columns, every local
  // column rewritten from its owner), projection sums, the replicated hierarchy's state
  double *rf_send = nullptr, *rf_recv = nullptr;
  int64_t rf_chunk = 0;
  double *pj_sums = nullptr, *pj_all = nullptr, *sub_w = nullptr;
  // Chebyshev-accelerated smoothing (WRMG_SMOOTH_CHEBYSHEV): lambda per level, direction / B r vectors
  bool cheb = false;
  std::vector<double> lam;
  std::vector<double *> cd, cbr;
};

namespace wrmg {
constexpr int kCoarseKronMax = 200;
extern std::atomic<int64_t> g_launches;  // kernels launched by this library (process-wide)
// Streaming multiprocessors of the current device (cached per device; 148 on B200).
int num_sms();
// Dynamic shared-memory opt-in (cudaFuncAttributeMaxDynamicSharedMemorySize) of a
// kernel on the current device, set once per (kernel, device) under a lock.
void smem_optin(const void *kernel, int bytes);
// Upper bound of the Krylov reduction blocks (multidot_blocks <= kDotBlocksMax).
constexpr int kDotBlocksMax = 1024;
// TMA tensor map of a waveform-major level vector: dims (NT, Lx, Ly), box (boxT, RW, RWy)
// (kernels_residual.cu; cached, thread-safe).  false if TMA cannot describe it.
bool umap_for(const double *u, int64_t NT, int Lx, int Ly, int boxT, int RW, CUtensorMap *out, int RWy = -1);
// kernel launchers (kernels_*.cu)
void launch_assemble_spatial(const Level &L, int k, const double *ref_dev, double kappa, cudaStream_t s);
void launch_patch_blocks(const Level &L, int nq, const Temporal &tm, cudaStream_t s);
void launch_coarse_G(Coarse &C, const Level &L, int nq, cudaStream_t s);  // GT, Gq from DinvT
void launch_batched_lu(double *A, int m, int batch, int32_t *piv, int32_t *info, cudaStream_t s);
void launch_inverse_and_G(const Level &L, const double *LU, int nq, cudaStream_t s);
void launch_coarse_blocks(const Level &L, Coarse &C, int nq, const Temporal &tm, cudaStream_t s);
void launch_coarse_inverse(Coarse &C, const double *LU, const Level &L, int nq, cudaStream_t s);
void launch_residual(const Level &L, int q, int N, const Temporal &tm, const double *u, const double *b,
                     double *r, bool u_is_zero, cudaStream_t s);
void launch_sweep(const Level &L, int q, int N, const double *r, double *u, double omega, cudaStream_t s);
void launch_restrict(const Level &coarse, int64_t nt, const double *rf, double *rc, cudaStream_t s);
void launch_prolong_add(const Level &coarse, int64_t nt, const double *ec, double *uf, cudaStream_t s);
void launch_coarse_solve(const Coarse &C, const Level &L, int q, int N, const double *r, double *x,
                         cudaStream_t s);
void launch_kron_setup(const Level &L, int nq, const Temporal &tm, double *scratch, cudaStream_t s);
void launch_kron_setup_coarse(const Level &L, Coarse &C, int nq, const Temporal &tm, double *scratch, cudaStream_t s);
bool launch_sweep_sym(const Level &L, int k, int q, int N, const double *r, double *u, double omega,
                      cudaStream_t s, const SweepLists *sl = nullptr);
bool launch_sweep_kron(const Level &L, int q, int N, const double *r, double *u, double omega, cudaStream_t s,
                       const SweepLists *sl = nullptr);
void launch_coarse_solve_kron(const Coarse &C, const Level &L, int q, int N, const double *r, double *x,
                              cudaStream_t s);
void launch_gather_classes(const Level &L, int32_t *scratch_i, double *scratch_d, cudaStream_t s);
bool launch_residual_mac(const Level &L, int k, int q, int N, const Temporal &tm, const double *u, const double *b,
                         double *r, cudaStream_t s);
bool plan_residual_mac(Level &L, int k, const std::vector<int32_t> &cnt, const std::vector<int32_t> &dI,
                       const std::vector<int32_t> &dJ, const std::vector<double> &m, const std::vector<double> &kk,
                       std::vector<int32_t> &gen_rows);
bool launch_residual_cls(const Level &L, int q, int N, const Temporal &tm, const double *u, const double *b,
                         double *r, cudaStream_t s);
void launch_rhs(const Level &L, int q, int N, const Temporal &tm, const double *fhat, double *b, cudaStream_t s);
void launch_fill_uniform(double *out, int64_t count, uint64_t first, uint64_t seed, cudaStream_t s);
// Krylov helpers
void launch_multidot(const double *const *V, int nv, const double *w, int64_t n, double *partials, int nblk,
                     cudaStream_t s);
int multidot_blocks(int64_t n);
void launch_cgs_update_dot(const double *const *V, int nv, double *w, const double *coef, int64_t n,
                           double *partials, int nblk, cudaStream_t s);
void launch_cgs_update_norm(const double *const *V, int nv, double *w, const double *coef, int64_t n,
                            double *partials, int nblk, cudaStream_t s);
void launch_reduce_partials(const double *partials, int nblk, int nv, double *out, cudaStream_t s);
void launch_multiaxpy(double *w, const double *const *V, const double *coef_dev, int nv, int64_t n, double sign,
                      cudaStream_t s);
void launch_scale(double *dst, const double *src, double a, int64_t n, cudaStream_t s);
void launch_cgs_step(double *kry, int j, int stage, cudaStream_t s);
// Chebyshev smoothing / initial state (kernels_cheb.cu)
void launch_cheb_update(int64_t n, double c1, double c2, const double *br, double *d, double *u, cudaStream_t s);
void launch_rhs_initial(const Level &L, int nq, int64_t NT, const double *phi0, const double *u0, double *b,
                        cudaStream_t s);
// strip partition (kernels_strip.cu)
void launch_cols(double *v, int Lx, int Ly, int64_t NT, int c0, int nc, double *buf, int mode, cudaStream_t s);
void launch_sum_chunks(const double *all, int nchunks, int64_t n, double *out, cudaStream_t s);
void launch_window(const double *src, int Lxs, int sc0, double *dst, int Lxd, int dc0, int Ly, int nc, int64_t NT,
                   cudaStream_t s);
}  // namespace wrmg
