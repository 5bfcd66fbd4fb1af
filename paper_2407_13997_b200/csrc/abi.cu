// C ABI (include/wrmg.h): setup of the space-time hierarchy, the smoother,
// V-cycle (H12) and FGMRES (H13) orchestration.  Every numerical step runs in
// the kernels of kernels_*.cu; this file only allocates, uploads integer plans
// and sequences launches on the context's stream.
#include <algorithm>
#include <climits>
#include <cmath>
#include <cstdlib>
#include <functional>
#include <mutex>

#include <nvtx3/nvToolsExt.h>  // header-only NVTX3: ranges per API call and kernel phase
#include <map>
#include <utility>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "comm.h"
#include "internal.h"
#include "lattice.h"
#include "ns.h"
#include "ns_kernels.h"
#include "plan.h"
#include "strip.h"
#include "sym.h"

using namespace wrmg;

namespace wrmg {
std::atomic<int64_t> g_launches{0};

int num_sms() {
  static std::atomic<int> cache[64] = {};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0) return 148;
  if (dev >= 64) {
    int v = 0;
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    return v > 0 ? v : 148;
  }
  int v = cache[dev].load(std::memory_order_relaxed);
  if (v <= 0) {
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0) v = 148;
    cache[dev].store(v, std::memory_order_relaxed);
  }
  return v;
}

void smem_optin(const void *kernel, int bytes) {
  static std::mutex mu;
  static std::map<std::pair<const void *, int>, int> done;  // (kernel, device) -> largest opt-in so far
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(mu);
  int &have = done[std::make_pair(kernel, dev)];
  if (bytes > have && cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes) == cudaSuccess)
    have = bytes;
}
bool hessenberg_eigenvalues(std::vector<double> &a, int n, std::vector<double> &wr, std::vector<double> &wi);
}

namespace {

thread_local std::string g_err;

struct Err {
  wrmg_status code;
  std::string msg;
};

#define CK(x)                                                                                  \
  do {                                                                                         \
    cudaError_t e_ = (x);                                                                      \
    if (e_ != cudaSuccess)                                                                     \
      throw Err{e_ == cudaErrorMemoryAllocation ? WRMG_E_OOM : WRMG_E_CUDA,                    \
                std::string(#x) + ": " + cudaGetErrorString(e_)};                              \
  } while (0)

// Guard bands (WRMG_GUARD=1; the stand-in for compute-sanitizer, which is closed on
// this GPU pool): every device allocation gets kGuard bytes of 0xFF on both sides --
// a NaN for doubles, -1 for indices, so an out-of-bounds read poisons the result the
// parity tests compare -- and dfree checks that no kernel wrote into them
// (wrmg_guard_violations() counts the corrupted bands).
constexpr size_t kGuard = 4096;
bool guard_on() {
  static const bool on = [] {
    const char *e = getenv("WRMG_GUARD");
    return e && e[0] == '1';
  }();
  return on;
}
std::mutex g_guard_mu;
std::map<void *, size_t> g_guard_sizes;  // user pointer -> user bytes
std::atomic<int64_t> g_guard_violations{0};

template <class T>
T *dalloc(size_t n) {
  void *p = nullptr;
  if (n == 0) n = 1;
  if (!guard_on()) {
    CK(cudaMalloc(&p, n * sizeof(T)));
    return (T *)p;
  }
  const size_t bytes = n * sizeof(T);
  CK(cudaMalloc(&p, bytes + 2 * kGuard));
  CK(cudaMemset(p, 0xFF, bytes + 2 * kGuard));
  CK(cudaStreamSynchronize(cudaStreamLegacy));  // the fill runs on the legacy stream: contexts on non-blocking streams are not ordered after it
  char *u = (char *)p + kGuard;
  std::lock_guard<std::mutex> lk(g_guard_mu);
  g_guard_sizes[u] = bytes;
  return (T *)u;
}
// Zero-initialised work vector (rows a kernel never writes -- e.g. a strip's
// non-owned columns -- then read as 0 instead of a recycled allocation's bytes).
template <class T>
T *dzalloc(size_t n) {
  T *p = dalloc<T>(n);
  CK(cudaMemset(p, 0, (n ? n : 1) * sizeof(T)));
  CK(cudaStreamSynchronize(cudaStreamLegacy));  // as above: the zeros must be in place before the context's stream uses p
  return p;
}

template <class T>
T *dupload(const std::vector<T> &v, cudaStream_t s) {
  T *p = dalloc<T>(v.size());
  if (!v.empty()) CK(cudaMemcpyAsync(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, s));
  return p;
}

void dfree(void *p) {
  if (!p) return;
  if (guard_on()) {
    size_t bytes = 0;
    {
      std::lock_guard<std::mutex> lk(g_guard_mu);
      auto it = g_guard_sizes.find(p);
      if (it != g_guard_sizes.end()) {
        bytes = it->second;
        g_guard_sizes.erase(it);
      }
    }
    if (bytes) {
      char *base = (char *)p - kGuard;
      std::vector<unsigned char> h(kGuard);
      for (const char *band : {base, base + kGuard + bytes}) {
        if (cudaMemcpy(h.data(), band, kGuard, cudaMemcpyDeviceToHost) != cudaSuccess) continue;
        for (unsigned char c : h)
          if (c != 0xFF) {
            ++g_guard_violations;
            fprintf(stderr, "wrmg guard: write outside a %zu-byte allocation\n", bytes);
            break;
          }
      }
      cudaFree(base);
      return;
    }
  }
  cudaFree(p);
}

wrmg_status fail(wrmg_ctx *ctx, const Err &e) {
  g_err = e.msg;
  if (ctx) ctx->err = e.msg;
  return e.code;
}

void check_launch() { CK(cudaGetLastError()); }

cudaEvent_t get_event(wrmg_ctx *c) {
  if (!c->prof_pool.empty()) {
    cudaEvent_t e = c->prof_pool.back();
    c->prof_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  CK(cudaEventCreate(&e));
  return e;
}

// Records a CUDA event pair around the launches issued in its scope (on the
// context's stream) when profiling is on, with the launches' algorithmic cost.
// NVTX range names of the kernel phases, "<class>_L<level>" (built once; no formatting per call)
const char *phase_name(int cls, int lvl) {
  static const char *kCls[] = {"residual", "sweep", "restrict", "prolong", "coarse", "krylov", "factor"};
  constexpr int kNc = (int)(sizeof(kCls) / sizeof(kCls[0])), kNl = 32;
  static const std::vector<std::string> names = [] {
    std::vector<std::string> v;
    for (int c2 = 0; c2 < kNc; ++c2)
      for (int l = 0; l < kNl; ++l) v.push_back(std::string(kCls[c2]) + "_L" + std::to_string(l));
    return v;
  }();
  if (cls < 0 || cls >= kNc || lvl < 0 || lvl >= kNl) return "phase";
  return names[(size_t)cls * kNl + lvl].c_str();
}

struct PScope {
  wrmg_ctx *c;
  int cls, lvl;
  double bytes, flops;
  cudaEvent_t a = nullptr, b = nullptr;
  PScope(wrmg_ctx *c_, int cls_, int lvl_, double bytes_, double flops_)
      : c(c_), cls(cls_), lvl(lvl_), bytes(bytes_), flops(flops_) {
    nvtxRangePushA(phase_name(cls, lvl));
    if (c->prof_on) {
      a = get_event(c);
      b = get_event(c);
      CK(cudaEventRecord(a, c->stream));
    }
  }
  ~PScope() {
    if (a) {
      cudaEventRecord(b, c->stream);
      c->prof_recs.push_back({cls, lvl, a, b, bytes, flops});
    }
    nvtxRangePop();
  }
};

double residual_bytes(const wrmg_ctx *c, int l) {
  return 24.0 * c->lv[l].nnode * c->nt + (c->ns ? 8.0 * c->lv[l].nvv * c->nt : 0.0);
}
double residual_flops(const wrmg_ctx *c, int l) {
  return 2.0 * (2 * c->nq + 1) * (double)c->lv[l].A.nnz * c->N;
}
double sweep_bytes(const wrmg_ctx *c, int l) {
  const Level &L = c->lv[l];
  // NS: every stored (patch, slab) inverse is streamed once per sweep
  return 24.0 * L.nfree * c->nt + (c->ns ? 8.0 * (double)L.npatch * c->N * L.mstride : 0.0);
}

NSGeom geom(const wrmg_ctx *c, const Level &L) {
  NSGeom g{};
  g.nx = L.nx;
  g.ny = L.ny;
  g.ku = c->k + 1;
  g.kp = c->k;
  g.Lux = L.Lux;
  g.Lpx = L.Lpx;
  g.nu = c->th_nu;
  g.np = c->th_np;
  g.Lu = L.Lu;
  g.Lp = L.Lp;
  g.ns = L.nnode;
  g.h = L.h;
  return g;
}

// Pressure mean removal per (slab, temporal node) of a level vector (H15, R19).
// Strips: the column sums over the owned pressure columns, all-gathered and summed in
// rank order (every rank subtracts bitwise the same mean).
void comm_call(wrmg_ctx *c, const std::function<void()> &f);
void ns_project(wrmg_ctx *c, const Level &L, double *v) {
  double *p = v + 2 * L.Lu * c->nt;
  if (!c->strip) {
    launch_ns_project(p, L.Lp, c->nt, c->proj, c->stream);
    return;
  }
  const StripInfo &S = L.stp;
  launch_ns_colsum_owned(p, L.Lpx, (int)(L.Lp / L.Lpx), S.own0, S.own1 - S.own0 + 1, c->nt, c->proj, c->pj_sums,
                         c->stream);
  comm_call(c, [&] { c->comm->allgather(c->pj_sums, c->pj_all, (size_t)c->nt, c->stream); });
  launch_ns_sub_gathered_mean(p, L.Lp, c->nt, c->pj_all, c->comm->nranks, L.gLp, c->pj_sums, c->stream);
}

void prof_residual(wrmg_ctx *c, int l, const double *u, const double *b, double *r, bool uzero,
                   const double *conv = nullptr) {
  PScope ps(c, WRMG_K_RESIDUAL, l, residual_bytes(c, l), uzero ? 0.0 : residual_flops(c, l));
  if (c->ns) {
    const Level &L = c->lv[l];
    launch_ns_residual(geom(c, L), c->q, c->N, c->tm, L.A, L.vvptr, conv ? conv : L.conv, L.con, u, b, r, c->stream);
    return;
  }
  launch_residual(c->lv[l], c->q, c->N, c->tm, u, b, r, uzero, c->stream);
}

void prof_sweep(wrmg_ctx *c, int l, const double *r, double *u, double om) {
  if (c->ns && c->lv[l].nswin < c->N) {  // slab windows: recompute each window's inverses, then sweep it
    const Level &L = c->lv[l];
    const double m = (double)c->nq * L.mp;
    for (int n0 = 0; n0 < c->N; n0 += L.nswin) {
      const int nw = std::min(L.nswin, c->N - n0);
      const double fr = (double)nw / c->N;
      {
        PScope pf(c, WRMG_K_FACTOR, l, 8.0 * (double)L.npatch * nw * L.mstride,
                  2.0 * m * m * m * (double)L.npatch * nw);
        launch_ns_factor(geom(c, L), c->q, c->N, c->tm, L.A, L.vvptr, L.conv, L.pnodes, L.npatch, L.mp, L.mstride,
                         L.nsinv, L.nsinfo, L.ppos, L.pvv, c->stream, n0, nw);
      }
      PScope ps(c, WRMG_K_SWEEP, l, sweep_bytes(c, l) * fr, c->sweep_flops[l] * fr);
      launch_ns_sweep(c->q, c->N, L.mp, L.npatch, L.mstride, L.pnodes, L.wnode, L.A, L.nsinv, r, u, om, c->stream,
                      n0, nw, L.nsxs);
    }
    if (!c->strip) ns_project(c, L, u);
    return;
  }
  PScope ps(c, WRMG_K_SWEEP, l, sweep_bytes(c, l), c->sweep_flops[l]);
  if (c->ns) {
    const Level &L = c->lv[l];
    launch_ns_sweep(c->q, c->N, L.mp, L.npatch, L.mstride, L.pnodes, L.wnode, L.A, L.nsinv, r, u, om, c->stream);
    if (!c->strip) ns_project(c, L, u);
    return;
  }
  if (c->use_kron && c->lv[l].coloured) {  // one pass per vertex colour: one addition per value and pass
    const Level &L = c->lv[l];
    for (int cc = 0; cc < 3; ++cc) {
      launch_sweep_sym(L, c->k, c->q, c->N, r, u, om, c->stream, &L.col[cc]);
      if (!launch_sweep_kron(L, c->q, c->N, r, u, om, c->stream, &L.col[cc]))
        throw Err{WRMG_E_UNSUPPORTED, "coloured scatter: no Kronecker sweep for this level"};
    }
    return;
  }
  if (c->use_kron) {
    const Level &L = c->lv[l];
    // WRMG_SWEEP_SIDE=1: boundary classes on a side stream, concurrently with the symmetric
    // class (C2, finest level only or every level: within noise of the serial order, 23.84-24.00
    // vs 23.90-23.91 ms per solve; coarser levels alone slower: off by default).  Read per
    // launch: the parity tests switch it.
    const char *se = getenv("WRMG_SWEEP_SIDE");
    const bool side = se && se[0] == '1';
    if (side && L.sym_ok && L.nsym > 0 && (L.kron_ngrp8 > 0 || L.kron_ncta > 0)) {
      // fork: the boundary classes on the side stream while the symmetric class runs
      if (!c->side) {
        CK(cudaStreamCreateWithFlags(&c->side, cudaStreamNonBlocking));
        CK(cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming));
      }
      CK(cudaEventRecord(c->ev_fork, c->stream));
      CK(cudaStreamWaitEvent(c->side, c->ev_fork, 0));
      if (!launch_sweep_kron(L, c->q, c->N, r, u, om, c->side))
        throw Err{WRMG_E_UNSUPPORTED, "no Kronecker sweep for the boundary classes"};
      launch_sweep_sym(L, c->k, c->q, c->N, r, u, om, c->stream);
      CK(cudaEventRecord(c->ev_join, c->side));
      CK(cudaStreamWaitEvent(c->stream, c->ev_join, 0));
      return;
    }
    const bool sym = launch_sweep_sym(L, c->k, c->q, c->N, r, u, om, c->stream);
    if (sym && L.kron_ngrp8 == 0 && L.kron_ncta == 0) return;  // every patch is in the symmetric class
    if (launch_sweep_kron(L, c->q, c->N, r, u, om, c->stream)) return;
  }
  launch_sweep(c->lv[l], c->q, c->N, r, u, om, c->stream);
}

void free_level(Level &L) {
  for (void *p : {(void *)L.A.rowptr, (void *)L.A.col, (void *)L.A.val, (void *)L.A.val2, (void *)L.con,
                  (void *)L.pnodes, (void *)L.ptype, (void *)L.wnode, (void *)L.type_rep, (void *)L.Dblk,
                  (void *)L.Dinv, (void *)L.G, (void *)L.piv, (void *)L.info, (void *)L.P.rowptr, (void *)L.P.col,
                  (void *)L.P.val, (void *)L.R.rowptr, (void *)L.R.col, (void *)L.R.val, (void *)L.vr, (void *)L.vz,
                  (void *)L.vt, (void *)L.kV, (void *)L.kVT, (void *)L.kS, (void *)L.ksig, (void *)L.cta_patch,
                  (void *)L.cta_type, (void *)L.rcls, (void *)L.cta_patch1, (void *)L.cta_type1,
                  (void *)L.goff, (void *)L.grp_patch8, (void *)L.grp_type8, (void *)L.vvptr, (void *)L.conv,
                  (void *)L.state, (void *)L.nsinv, (void *)L.nsxs, (void *)L.nsinfo, (void *)L.ppos, (void *)L.pvv, (void *)L.hx[0],
                  (void *)L.hx[1],
                  (void *)L.hx[2], (void *)L.hx[3], (void *)L.gen_rows, (void *)L.sym_nodes,
                  (void *)L.tile_patch, (void *)L.sym_single, (void *)L.tgeo_dev})
    dfree(p);
  for (auto &S : L.col)
    for (void *p : {(void *)S.cta_patch, (void *)S.cta_type, (void *)S.grp_patch8, (void *)S.grp_type8,
                    (void *)S.sym_list})
      dfree(p);
}

void validate(const wrmg_mesh *mesh, int degree, int q, int nslabs, double dt) {
  if (!mesh) throw Err{WRMG_E_INVALID, "mesh is NULL"};
  if (degree < 1 || degree > 3) throw Err{WRMG_E_UNSUPPORTED, "degree must be 1..3"};
  if (q < 0 || q > 3) throw Err{WRMG_E_UNSUPPORTED, "q must be 0..3"};
  if (nslabs < 1) throw Err{WRMG_E_INVALID, "nslabs must be >= 1"};
  if (!(dt > 0)) throw Err{WRMG_E_INVALID, "dt must be > 0"};
  if (mesh->gnx < 1 || mesh->gny < 1 || !(mesh->h > 0)) throw Err{WRMG_E_INVALID, "bad mesh size"};
  if (mesh->x0 < 0 || mesh->nx < 0 || mesh->x0 + mesh->nx > mesh->gnx) throw Err{WRMG_E_INVALID, "bad strip"};
  int64_t L = (int64_t)(degree * mesh->gnx + 1) * (degree * mesh->gny + 1);
  if (L > (int64_t)INT32_MAX / 8) throw Err{WRMG_E_UNSUPPORTED, "lattice too large for int32 node ids"};
}

// Copy the residual stencil-class tables of a level to the host (kernel parameter).
void gather_stencil(wrmg_ctx *c, Level &L) {
  const int nc = (int)L.h_cls_rep.size();
  L.stencil_ok = false;
  if (nc == 0 || nc > kStencilMaxC) return;
  int32_t *si = dalloc<int32_t>((size_t)2 * nc + 2 * nc * kStencilMaxE);
  double *sd = dalloc<double>((size_t)2 * nc * kStencilMaxE);
  CK(cudaMemcpyAsync(si, L.h_cls_rep.data(), nc * sizeof(int32_t), cudaMemcpyHostToDevice, c->stream));
  launch_gather_classes(L, si, sd, c->stream);
  check_launch();
  std::vector<int32_t> hi((size_t)2 * nc + 2 * nc * kStencilMaxE);
  std::vector<double> hd((size_t)2 * nc * kStencilMaxE);
  CK(cudaMemcpyAsync(hi.data(), si, hi.size() * sizeof(int32_t), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaMemcpyAsync(hd.data(), sd, hd.size() * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  dfree(si);
  dfree(sd);
  StencilTab &T = L.stencil;
  std::memset(&T, 0, sizeof(T));
  T.ncls = nc;
  const int32_t *cnt = hi.data() + nc, *dI = cnt + nc, *dJ = dI + nc * kStencilMaxE;
  const int RW = 8 + 2 * c->k;  // residual tile (kernels_residual.cu) + k-wide halo
  for (int k2 = 0; k2 < nc; ++k2) {
    if (((cnt[k2] + 3) & ~3) > kStencilMaxE) return;
    T.cnt[k2] = (cnt[k2] + 3) & ~3;  // zero entries pad the loop to a multiple of 4
    for (int e = 0; e < cnt[k2]; ++e) {
      T.off[k2][e] = (dJ[k2 * kStencilMaxE + e] * RW + dI[k2 * kStencilMaxE + e]) * 32 * c->nq;
      T.m[k2][e] = hd[k2 * kStencilMaxE + e];
      T.kk[k2][e] = hd[nc * kStencilMaxE + k2 * kStencilMaxE + e];
    }
  }
  std::vector<int64_t> go((size_t)kStencilMaxC * kStencilMaxE, 0);
  for (int k2 = 0; k2 < nc; ++k2)
    for (int e = 0; e < cnt[k2]; ++e)
      go[k2 * kStencilMaxE + e] =
          ((int64_t)dJ[k2 * kStencilMaxE + e] * L.Lx + dI[k2 * kStencilMaxE + e]) * c->nt;
  if (!L.goff) L.goff = dalloc<int64_t>(go.size());
  CK(cudaMemcpy(L.goff, go.data(), go.size() * sizeof(int64_t), cudaMemcpyHostToDevice));
  L.stencil_ok = true;
  // macro-block residual: interior classes per row type, fix-up list of the other rows
  std::vector<int32_t> vc(cnt, cnt + nc), vI(dI, dI + nc * kStencilMaxE), vJ(dJ, dJ + nc * kStencilMaxE), gen;
  std::vector<double> vm(hd.begin(), hd.begin() + nc * kStencilMaxE), vk(hd.begin() + nc * kStencilMaxE, hd.end());
  L.mac_ok = plan_residual_mac(L, c->k, vc, vI, vJ, vm, vk, gen);
  dfree(L.gen_rows);
  L.gen_rows = nullptr;
  L.ngen_rows = 0;
  if (L.mac_ok && !gen.empty()) {
    L.gen_rows = dalloc<int32_t>(gen.size());
    CK(cudaMemcpy(L.gen_rows, gen.data(), gen.size() * sizeof(int32_t), cudaMemcpyHostToDevice));
    L.ngen_rows = (int64_t)gen.size();
  }
}


// ------------------------------------------------------------ strip partition
// Halo updates of a level vector (strip.h for the columns).
void comm_call(wrmg_ctx *c, const std::function<void()> &f) {
  try {
    f();
  } catch (const std::string &m) {
    throw Err{WRMG_E_NCCL, m};
  }
}

// The lattice fields of a level vector: heat one lattice; Navier-Stokes u_x, u_y
// (velocity lattice, degree k + 1) and p (pressure lattice, degree k), each with its
// own column bookkeeping (ns.h: plan_ns_strip_level).
struct FieldView {
  int64_t off;  // first double of the field in the level vector
  int Lx, Ly, k;
  int64_t goff;  // global sid of the field's first node (canonical ids)
  const StripInfo *S;
};
int level_fields(const wrmg_ctx *c, const Level &L, FieldView *f) {
  if (!c->ns) {
    f[0] = {0, L.Lx, L.Ly, c->k, 0, &L.st};
    return 1;
  }
  const int ku = c->k + 1, kp = c->k;
  const int Lpy = (int)(L.Lp / L.Lpx);
  const int64_t GLu = (int64_t)(ku * L.st.gnx + 1) * L.Ly;
  f[0] = {0, L.Lux, L.Ly, ku, 0, &L.st};
  f[1] = {L.Lu * c->nt, L.Lux, L.Ly, ku, GLu, &L.st};
  f[2] = {2 * L.Lu * c->nt, L.Lpx, Lpy, kp, 2 * GLu, &L.stp};
  return 3;
}
// doubles of one halo buffer (k ghost columns of every field)
int64_t halo_doubles(const wrmg_ctx *c, const Level &L) {
  FieldView f[3];
  const int nf = level_fields(c, L, f);
  int64_t n = 0;
  for (int i = 0; i < nf; ++i) n += (int64_t)f[i].Ly * f[i].k * c->nt;
  return n;
}

// mode 0: pack the columns (c0, nc) of every field into buf; 1: unpack; 2: unpack-add
size_t halo_cols(wrmg_ctx *c, Level &L, double *v, bool left_side, bool ghosts, double *buf, int mode) {
  FieldView f[3];
  const int nf = level_fields(c, L, f);
  size_t o = 0;
  for (int i = 0; i < nf; ++i) {
    const StripInfo &S = *f[i].S;
    const int c0 = ghosts ? (left_side ? S.lg0 : S.rg0) : (left_side ? S.sl0 : S.sr0);
    const int nc = ghosts ? (left_side ? S.nlg : S.nrg) : (left_side ? S.nsl : S.nsr);
    launch_cols(v + f[i].off, f[i].Lx, f[i].Ly, c->nt, c0, nc, buf + o, mode, c->stream);
    o += (size_t)f[i].Ly * nc * c->nt;
  }
  return o;
}

// ghosts <- owners (both sides)
void halo_forward(wrmg_ctx *c, Level &L, double *v) {
  const size_t nL = halo_cols(c, L, v, true, false, L.hx[0], 0);
  const size_t nR = halo_cols(c, L, v, false, false, L.hx[2], 0);
  comm_call(c, [&] { c->comm->exchange(L.hx[0], L.hx[1], nL, L.hx[2], L.hx[3], nR, c->stream); });
  halo_cols(c, L, v, true, true, L.hx[1], 1);
  halo_cols(c, L, v, false, true, L.hx[3], 1);
}

// owners += ghosts of the neighbours (both sides)
void halo_reverse_add(wrmg_ctx *c, Level &L, double *v) {
  const size_t nL = halo_cols(c, L, v, true, true, L.hx[0], 0);
  const size_t nR = halo_cols(c, L, v, false, true, L.hx[2], 0);
  comm_call(c, [&] { c->comm->exchange(L.hx[0], L.hx[1], nL, L.hx[2], L.hx[3], nR, c->stream); });
  halo_cols(c, L, v, true, false, L.hx[1], 2);
  halo_cols(c, L, v, false, false, L.hx[3], 2);
}

// Zero every column this rank does not own: the ghost columns and, on ranks > 0, the
// local lattice's first column (one cell left of the left ghosts; never refreshed --
// with Neumann boundaries it is a free row, so dot products must not see it).
void zero_ghosts(wrmg_ctx *c, Level &L, double *v) {
  FieldView f[3];
  const int nf = level_fields(c, L, f);
  for (int i = 0; i < nf; ++i) {
    const StripInfo &S = *f[i].S;
    double *p = v + f[i].off;
    if (S.own0 > 0) launch_cols(p, f[i].Lx, f[i].Ly, c->nt, 0, S.own0, nullptr, 3, c->stream);
    if (S.own1 + 1 < f[i].Lx)
      launch_cols(p, f[i].Lx, f[i].Ly, c->nt, S.own1 + 1, f[i].Lx - S.own1 - 1, nullptr, 3, c->stream);
  }
}

// Navier-Stokes strips: every local column of v (owned, ghost and the overlap cells
// beyond) rewritten from its owner -- all-gather of the owned columns.  The
// linearisation state needs it: the Vanka blocks of the owned patches integrate over
// cells up to two columns of cells beyond the owned ones (ns.h).
void state_refresh(wrmg_ctx *c, Level &L, double *v) {
  FieldView f[3];
  const int nf = level_fields(c, L, f);
  cudaStream_t s = c->stream;
  size_t o = 0;
  for (int i = 0; i < nf; ++i) {
    const StripInfo &S = *f[i].S;
    const int nown = S.own1 - S.own0 + 1;
    launch_cols(v + f[i].off, f[i].Lx, f[i].Ly, c->nt, S.own0, nown, c->rf_send + o, 0, s);
    o += (size_t)f[i].Ly * nown * c->nt;
  }
  if ((int64_t)o > c->rf_chunk) throw Err{WRMG_E_INVALID, "state refresh: chunk overflow"};
  comm_call(c, [&] { c->comm->allgather(c->rf_send, c->rf_recv, (size_t)c->rf_chunk, s); });
  for (int q = 0; q < c->comm->nranks; ++q) {
    size_t oq = 0;
    for (int i = 0; i < nf; ++i) {
      const StripInfo &S = *f[i].S;
      const int k = f[i].k, x0q = q * S.nx;
      const int g0q = q == 0 ? 0 : k * x0q + 1, g1q = k * (x0q + S.nx), nq = g1q - g0q + 1;
      const int ov0 = std::max(g0q, S.G0), ov1 = std::min(g1q, S.G0 + f[i].Lx - 1);
      if (ov0 <= ov1)
        launch_window(c->rf_recv + (int64_t)q * c->rf_chunk + oq, nq, ov0 - g0q, v + f[i].off, f[i].Lx, ov0 - S.G0,
                      f[i].Ly, ov1 - ov0 + 1, c->nt, s);
      oq += (size_t)f[i].Ly * nq * c->nt;
    }
  }
}

// One additive sweep on a strip: owned patches add into owned and right-ghost
// columns; the ghost sums are returned to their owners, then ghosts refreshed.
void ns_project(wrmg_ctx *c, const Level &L, double *v);

void sweep_strip(wrmg_ctx *c, int l, const double *r, double *u, double om) {
  Level &L = c->lv[l];
  zero_ghosts(c, L, u);
  prof_sweep(c, l, r, u, om);
  halo_reverse_add(c, L, u);
  if (c->ns) ns_project(c, L, u);  // the pressure mean of the summed update (every rank subtracts the same)
  halo_forward(c, L, u);
}

// Coarsest level: all-gather the owned columns, replicated exact solve of the
// global coarsest problem (H11), local window (owned + ghosts) back.
void coarse_strip(wrmg_ctx *c, const double *r, double *z) {
  Level &L0 = c->lv[0];
  Level &G = c->gco;
  const StripInfo &S = L0.st;
  cudaStream_t s = c->stream;
  const int k = c->k, nx0 = S.nx;
  launch_cols(const_cast<double *>(r), L0.Lx, L0.Ly, c->nt, S.own0, S.own1 - S.own0 + 1, c->gsend, 0, s);
  comm_call(c, [&] { c->comm->allgather(c->gsend, c->grecv, (size_t)c->gchunk, s); });
  for (int q = 0; q < S.nranks; ++q) {
    const int x0q = q * nx0;
    const int g0 = q == 0 ? 0 : k * x0q + 1, g1 = k * (x0q + nx0);
    launch_window(c->grecv + (int64_t)q * c->gchunk, g1 - g0 + 1, 0, c->gr, G.Lx, g0, G.Ly, g1 - g0 + 1, c->nt, s);
  }
  {
    const Coarse &C = c->coarse;
    PScope ps(c, WRMG_K_COARSE, 0, 16.0 * C.nfree * c->nt + 8.0 * G.nnode * c->nt,
              2.0 * c->N * ((double)C.m * C.m + (double)C.m * C.mp));
    if (c->coarse_kron)
      launch_coarse_solve_kron(C, G, c->q, c->N, c->gr, c->gz, s);
    else
      launch_coarse_solve(C, G, c->q, c->N, c->gr, c->gz, s);
  }
  launch_window(c->gz, G.Lx, S.G0, z, L0.Lx, 0, L0.Ly, L0.Lx, c->nt, s);
}

bool sym_disabled() {  // WRMG_SWEEP_SYM=0: every class through kernels_kron.cu (A/B)
  const char *e = getenv("WRMG_SWEEP_SYM");
  return e && e[0] == '0';
}
bool tiles_disabled() {  // WRMG_SWEEP_TILES=1: the 2 x 2 tiled symmetric sweep (measured slower)
  const char *e = getenv("WRMG_SWEEP_TILES");
  return !(e && e[0] == '1');
}

// 2 x 2 tiles of symmetric-class patches (even vertex coordinates) for the tiled
// sweep; every tile must have the representative's union geometry, else the tiled
// form is not used on this level.
void plan_sym_tiles(const PlanLevel &P, int k, int cls, int mp, const std::vector<int32_t> &sn, Level &L,
                    cudaStream_t s) {
  const int nvx = P.nx + 1;
  std::vector<int32_t> at((size_t)nvx * (P.ny + 1), -1);  // vertex -> index in the symmetric list
  {
    int32_t q = 0;
    for (int64_t p = 0; p < P.npatch; ++p)
      if (P.ptype[p] == cls) at[P.pvert[p]] = q++;
  }
  std::vector<int32_t> tiles, single;
  std::vector<uint8_t> used(L.nsym, 0);
  TileGeom G{};
  bool have = false, ok = !tiles_disabled();
  for (int vj = 0; ok && vj + 1 <= P.ny; vj += 2)
    for (int vi = 0; ok && vi + 1 <= P.nx; vi += 2) {
      const int32_t q[4] = {at[vj * nvx + vi], at[vj * nvx + vi + 1], at[(vj + 1) * nvx + vi],
                            at[(vj + 1) * nvx + vi + 1]};
      if (q[0] < 0 || q[1] < 0 || q[2] < 0 || q[3] < 0) continue;
      const int64_t base = (int64_t)k * vj * P.Lx + k * vi;
      TileGeom T{};
      for (int w = 0; w < 4; ++w)
        for (int j = 0; j < mp; ++j) {
          const int32_t o = (int32_t)(sn[(size_t)q[w] * mp + j] - base);
          int u = 0;
          while (u < T.nu && T.off[u] != o) ++u;
          if (u == T.nu) {
            if (T.nu == kTileMaxU) { ok = false; break; }
            T.off[T.nu++] = o;
          }
          if (T.cnt[u] == 4) { ok = false; break; }
          T.src[u][T.cnt[u]++] = (int16_t)(w * mp + j);
        }
      if (!ok) break;
      if (!have) {
        for (int u = 0; u < T.nu; ++u) {  // interior: the node's entity vertices all lie in the tile
          const int64_t g = base + T.off[u];
          int ei[3], ej[3];
          const int ne = entity_vertices(k, (int)(g % P.Lx), (int)(g / P.Lx), ei, ej);
          bool in = true;
          for (int e = 0; e < ne; ++e) in = in && ei[e] >= vi && ei[e] <= vi + 1 && ej[e] >= vj && ej[e] <= vj + 1;
          T.interior[u] = in;
        }
        G = T;
        have = true;
      } else {
        bool same = T.nu == G.nu;
        for (int u = 0; same && u < T.nu; ++u) {
          same = T.off[u] == G.off[u] && T.cnt[u] == G.cnt[u];
          for (int e = 0; same && e < T.cnt[u]; ++e) same = T.src[u][e] == G.src[u][e];
        }
        if (!same) { ok = false; break; }
      }
      for (int w = 0; w < 4; ++w) {
        tiles.push_back(q[w]);
        used[q[w]] = 1;
      }
    }
  if (!ok || !have) {
    tiles.clear();
    std::fill(used.begin(), used.end(), 0);
  }
  for (int64_t q = 0; q < L.nsym; ++q)
    if (!used[q]) single.push_back((int32_t)q);
  L.ntile = (int64_t)tiles.size() / 4;
  L.nsingle = (int64_t)single.size();
  L.tgeo = (ok && have) ? G : TileGeom{};
  if (L.ntile) {
    L.tile_patch = dupload(tiles, s);
    L.tgeo_dev = dupload(std::vector<TileGeom>{L.tgeo}, s);
  }
  if (L.nsingle) L.sym_single = dupload(single, s);
}



// Symmetry-reduced sweep coefficients of the interior class from the assembled M, kappa K.
void sym_setup(wrmg_ctx *c, Level &L) {
  const int mps = (int)std::lround(std::sqrt((double)L.sym_pos.size()));
  int64_t lo = INT64_MAX, hi = -1;
  for (int64_t e : L.sym_pos)
    if (e >= 0) {
      lo = std::min(lo, e);
      hi = std::max(hi, e);
    }
  if (hi < 0) throw Err{WRMG_E_INVALID, "symmetric patch block has no entries"};
  std::vector<double> mv(hi - lo + 1), kv(hi - lo + 1);
  CK(cudaMemcpy(mv.data(), L.A.val + lo, mv.size() * sizeof(double), cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(kv.data(), L.A.val2 + lo, kv.size() * sizeof(double), cudaMemcpyDeviceToHost));
  std::vector<double> Mp((size_t)mps * mps, 0.0), Kp((size_t)mps * mps, 0.0);
  for (size_t e = 0; e < L.sym_pos.size(); ++e)
    if (L.sym_pos[e] >= 0) {
      Mp[e] = mv[L.sym_pos[e] - lo];
      Kp[e] = kv[L.sym_pos[e] - lo];
    }
  if (!sym_factor(c->k, Mp.data(), Kp.data(), c->tm, &L.symtab))
    throw Err{WRMG_E_SINGULAR, "symmetry-reduced patch factorisation failed"};
}

// Numeric part of setup / linearisation: H1, H4, H5 on every level + coarse block.
void factor_all(wrmg_ctx *c) {
  cudaStream_t s = c->stream;
  for (auto &L : c->lv) {
    launch_assemble_spatial(L, c->k, c->ref_dev, c->co.kappa, s);
    check_launch();
    launch_patch_blocks(L, c->nq, c->tm, s);
    check_launch();
    const int m = c->nq * L.mp;
    double *LU = dalloc<double>((size_t)L.ntypes * m * m);
    CK(cudaMemcpyAsync(LU, L.Dblk, (size_t)L.ntypes * m * m * sizeof(double), cudaMemcpyDeviceToDevice, s));
    launch_batched_lu(LU, m, L.ntypes, L.piv, L.info, s);
    check_launch();
    launch_inverse_and_G(L, LU, c->nq, s);
    check_launch();
    CK(cudaStreamSynchronize(s));
    dfree(LU);
    if (c->use_kron) {
      double *scr = dalloc<double>((size_t)L.ntypes * 3 * L.mp * L.mp);
      launch_kron_setup(L, c->nq, c->tm, scr, s);
      check_launch();
      CK(cudaStreamSynchronize(s));
      dfree(scr);
    }
    if (L.sym_ok) sym_setup(c, L);
    gather_stencil(c, L);
  }
  if (c->sub) return;  // the replicated hierarchy factored its own levels and coarse solve
  Coarse &C = c->coarse;
  Level &L0 = c->strip ? c->gco : c->lv[0];  // strips: the replicated global coarsest level
  if (c->strip) {
    launch_assemble_spatial(L0, c->k, c->ref_dev, c->co.kappa, s);
    check_launch();
  }
  launch_coarse_blocks(L0, C, c->nq, c->tm, s);
  check_launch();
  double *LU = dalloc<double>((size_t)C.m * C.m);
  CK(cudaMemcpyAsync(LU, C.Dblk, (size_t)C.m * C.m * sizeof(double), cudaMemcpyDeviceToDevice, s));
  if (C.m >= kGJMinM) {  // blocked Gauss-Jordan inverse (kernels_gj.cu)
    double *scr = dalloc<double>(gj_scratch_doubles(C.m, 1));
    launch_gj_inverse_batched(LU, C.m, 1, C.piv, C.info, C.DinvT, scr, s);
    check_launch();
    launch_coarse_G(C, L0, c->nq, s);
    check_launch();
    CK(cudaStreamSynchronize(s));
    dfree(scr);
  } else {
    launch_batched_lu(LU, C.m, 1, C.piv, C.info, s);
    check_launch();
    launch_coarse_inverse(C, LU, L0, c->nq, s);
    check_launch();
  }
  CK(cudaStreamSynchronize(s));
  dfree(LU);
  if (c->coarse_kron) {
    double *scr = dalloc<double>((size_t)3 * C.mp * C.mp);
    launch_kron_setup_coarse(L0, C, c->nq, c->tm, scr, s);
    check_launch();
    CK(cudaStreamSynchronize(s));
    dfree(scr);
  }
  // singular pivots (R10)
  c->err_level = c->err_patch = c->err_slab = -1;
  for (size_t l = 0; l < c->lv.size(); ++l) {
    Level &L = c->lv[l];
    std::vector<int32_t> info(L.ntypes);
    CK(cudaMemcpy(info.data(), L.info, L.ntypes * sizeof(int32_t), cudaMemcpyDeviceToHost));
    for (int t = 0; t < L.ntypes; ++t)
      if (info[t]) {
        c->err_level = (int)l;
        c->err_patch = L.h_type_rep[t];
        c->err_slab = -1;  // time-invariant block: every slab
        throw Err{WRMG_E_SINGULAR, "singular patch block (level " + std::to_string(l) + ", patch " +
                                       std::to_string(L.h_type_rep[t]) + ", column " + std::to_string(info[t]) + ")"};
      }
  }
  int32_t ci = 0;
  CK(cudaMemcpy(&ci, C.info, sizeof(int32_t), cudaMemcpyDeviceToHost));
  if (ci) {
    c->err_level = 0;
    c->err_patch = -1;
    throw Err{WRMG_E_SINGULAR, "singular coarse block (column " + std::to_string(ci) + ")"};
  }
}


double estimate_lambda(wrmg_ctx *c, int l);

// Navier-Stokes linearisation at the finest-level state W (NULL = zero state):
// inject W to every level (R13), assemble R N(W) (H1), invert every (patch, slab)
// block (H4, H5) and the pinned coarse slab blocks (H11).  Synchronises.
void state_refresh(wrmg_ctx *c, Level &L, double *v);

// Singular (patch, slab) blocks of levels >= l0 -> WRMG_E_SINGULAR with the location.
void check_ns_patch_info(wrmg_ctx *c, int l0) {
  c->err_level = c->err_patch = c->err_slab = -1;
  for (int l = l0; l < (int)c->lv.size(); ++l) {
    Level &L = c->lv[l];
    std::vector<int32_t> info((size_t)L.npatch * c->N);
    CK(cudaMemcpy(info.data(), L.nsinfo, info.size() * sizeof(int32_t), cudaMemcpyDeviceToHost));
    for (size_t e = 0; e < info.size(); ++e)
      if (info[e]) {
        c->err_level = l;
        c->err_patch = (int)(e / c->N);
        c->err_slab = (int)(e % c->N);
        throw Err{WRMG_E_SINGULAR, "singular Vanka patch block (level " + std::to_string(l) + ", patch " +
                                       std::to_string(c->err_patch) + ", slab " + std::to_string(c->err_slab) + ")"};
      }
  }
}

void factor_all_ns(wrmg_ctx *c, const double *W) {
  cudaStream_t s = c->stream;
  const int nl = (int)c->lv.size();
  const double *Wl = W;
  if (c->strip && W) {  // strips: a copy of the state with every local column from its owner
    Level &F = c->lv.back();
    CK(cudaMemcpyAsync(F.state, W, F.nnode * c->nt * sizeof(double), cudaMemcpyDeviceToDevice, s));
    state_refresh(c, F, F.state);
    Wl = F.state;
  }
  for (int l = nl - 1; l >= 0; --l) {
    Level &L = c->lv[l];
    if (l < nl - 1 && W) {
      if (c->strip) {  // owned coarse columns from owned fine columns, then the refresh
        const Level &F = c->lv[l + 1];
        const NSInjMap m{2 * L.st.G0 - F.st.G0, 2 * L.stp.G0 - F.stp.G0, F.st.own0, F.st.own1, F.stp.own0, F.stp.own1};
        launch_ns_inject(geom(c, L), geom(c, F), c->nt, Wl, L.state, s, &m);
        state_refresh(c, L, L.state);
      } else {
        launch_ns_inject(geom(c, L), geom(c, c->lv[l + 1]), c->nt, Wl, L.state, s);
      }
      Wl = L.state;
    }
    launch_ns_assemble_conv(geom(c, L), c->nt, c->co.reynolds, true, L.A, L.vvptr, W ? Wl : nullptr, L.conv,
                            c->th_T, s);
    check_launch();
    if (l >= 1 || nl == 1 || c->strip) {
      const double m = (double)c->nq * L.mp;
      PScope ps(c, WRMG_K_FACTOR, l, 8.0 * (double)L.npatch * c->N * L.mstride,
                2.0 * m * m * m * (double)L.npatch * c->N);
      // slab windows: every window factored once here for the singularity check (the sweeps
      // recompute them); a stored level is one window
      for (int n0 = 0; n0 < c->N; n0 += L.nswin)
        launch_ns_factor(geom(c, L), c->q, c->N, c->tm, L.A, L.vvptr, L.conv, L.pnodes, L.npatch, L.mp, L.mstride,
                         L.nsinv, L.nsinfo, L.ppos, L.pvv, s, n0, std::min(L.nswin, c->N - n0));
      check_launch();
    }
  }
  if (c->strip) {
    // the replicated hierarchy (levels below the partitioned ones): its finest level's
    // state by injection of the owned columns of level 0, summed over ranks in rank order
    const double *Ws = nullptr;
    if (W) {
      const Level &T = c->sub->lv.back(), &L0 = c->lv[0];
      const int64_t ng = T.nnode * c->nt;
      const NSInjMap m{-L0.st.G0, -L0.stp.G0, L0.st.own0, L0.st.own1, L0.stp.own0, L0.stp.own1};
      launch_ns_inject(geom(c->sub, T), geom(c, L0), c->nt, Wl, c->sub_part, s, &m);
      comm_call(c, [&] { c->comm->allgather(c->sub_part, c->sub_all, (size_t)ng, s); });
      launch_sum_chunks(c->sub_all, c->comm->nranks, ng, c->sub_w, s);
      Ws = c->sub_w;
    }
    factor_all_ns(c->sub, Ws);
    CK(cudaStreamSynchronize(s));
    check_ns_patch_info(c, 0);
    if (c->cheb)
      for (int l = 0; l < nl; ++l) c->lam[l] = estimate_lambda(c, l);
    return;
  }
  Coarse &C = c->coarse;
  Level &L0 = c->lv[0];
  launch_ns_coarse_blocks(geom(c, L0), c->q, c->N, c->tm, L0.A, L0.vvptr, L0.conv, C.nodes, C.mp, C.pin, C.nsD, s);
  check_launch();
  {
    PScope ps(c, WRMG_K_FACTOR, 0, 16.0 * (double)c->N * C.m * C.m, 2.0 * (double)C.m * C.m * C.m * c->N);
    if (C.m >= kGJMinM) {
      double *scr = dalloc<double>(gj_scratch_doubles(C.m, c->N));
      launch_gj_inverse_batched(C.nsD, C.m, c->N, C.nspiv, C.nsinfo, C.nsinvT, scr, s);
      check_launch();
      CK(cudaStreamSynchronize(s));
      dfree(scr);
    } else {
      launch_batched_lu(C.nsD, C.m, c->N, C.nspiv, C.nsinfo, s);
      check_launch();
      launch_lu_inverse_batched(C.nsD, C.nspiv, C.m, c->N, C.nsinvT, s);
      check_launch();
    }
  }
  launch_ns_coarse_H(c->q, c->N, C.mp, C.pin, C.nodes, C.sid2c, L0.A, C.nsinvT, C.nsH, C.nsG, s);
  check_launch();
  CK(cudaStreamSynchronize(s));
  check_ns_patch_info(c, nl == 1 ? 0 : 1);
  std::vector<int32_t> ci(c->N);
  CK(cudaMemcpy(ci.data(), C.nsinfo, c->N * sizeof(int32_t), cudaMemcpyDeviceToHost));
  for (int n = 0; n < c->N; ++n)
    if (ci[n]) {
      c->err_level = 0;
      c->err_slab = n;
      throw Err{WRMG_E_SINGULAR, "singular coarse slab block (slab " + std::to_string(n) + ")"};
    }
  if (c->cheb)  // the relaxed operator changed: new Chebyshev intervals (R-cheb)
    for (int l = 1; l < nl; ++l) c->lam[l] = estimate_lambda(c, l);
}

// Uniform strips x0 = rank * nx: the transport.
void make_strip_comm(wrmg_ctx *c) {
  const int P = c->co.nranks, r = c->co.rank;
  if (r < 0 || r >= P || c->mesh.nx * P != c->mesh.gnx || c->mesh.x0 != r * c->mesh.nx)
    throw Err{WRMG_E_INVALID, "strips: need nx * nranks = gnx and x0 = rank * nx"};
  std::string e;
  c->comm = c->co.loopback_hub ? make_loop_comm(c->co.loopback_hub, r, P, e)
                               : make_nccl_comm(c->co.nccl_unique_id, r, P, e);
  if (!c->comm) throw Err{WRMG_E_NCCL, e};
}

// Hierarchy of Taylor-Hood levels (problem == WRMG_NAVIER_STOKES).
// Stored Vanka inverses (m^2 doubles per (patch, slab)): levels whose store does not fit
// the memory budget keep a window of W slabs only and recompute it inside every sweep
// ("slab windows"): the budget is 92 % of the free device memory less 8 GB
// (a later FGMRES(30) allocates 62 more vectors; lower the budget with WRMG_NS_STORE_GB
// when they must fit beside a large store); while the stores exceed it, the level with
// the largest store halves its window.  WRMG_NS_WINDOW=<W> windows every stored level at W
// slabs (tests), WRMG_NS_STORE_GB=<GB> sets the budget.
void ns_slab_windows(wrmg_ctx *c) {
  std::vector<Level *> ls;
  for (auto &L : c->lv)
    if (L.nsinfo) ls.push_back(&L);
  for (Level *L : ls) L->nswin = c->N;
  auto per_slab = [&](const Level *L) { return 8.0 * (double)L->npatch * (double)L->mstride; };
  if (const char *e = getenv("WRMG_NS_WINDOW")) {
    const int w = atoi(e);
    if (w > 0)
      for (Level *L : ls) L->nswin = std::min(w, c->N);
  } else {
    size_t fr = 0, tot = 0;
    CK(cudaMemGetInfo(&fr, &tot));
    double budget = 0.92 * (double)fr - 8e9;
    if (const char *e = getenv("WRMG_NS_STORE_GB")) budget = atof(e) * 1e9;
    auto total = [&] {
      double t = 0.0;
      for (Level *L : ls) t += per_slab(L) * L->nswin;
      return t;
    };
    while (total() > budget) {
      Level *big = nullptr;
      for (Level *L : ls)
        if (L->nswin > 1 && (!big || per_slab(L) * L->nswin > per_slab(big) * big->nswin)) big = L;
      if (!big) throw Err{WRMG_E_OOM, "Vanka inverses: one slab per level does not fit the device"};
      big->nswin = (big->nswin + 1) / 2;
    }
  }
  for (Level *L : ls) {
    L->nsinv = dalloc<double>((size_t)L->npatch * L->nswin * L->mstride);
    if (L->nswin < c->N) L->nsxs = dzalloc<double>((size_t)L->npatch * c->nq * L->mp);
  }
}

void setup_ns(wrmg_ctx *c) {
  cudaStream_t s = c->stream;
  if (c->k > 2) throw Err{WRMG_E_UNSUPPORTED, "Navier-Stokes: degree must be 1 (P2-P1) or 2 (P3-P2)"};
  if (!(c->co.reynolds > 0)) throw Err{WRMG_E_INVALID, "Reynolds number must be > 0"};
  if (c->co.bc != WRMG_BC_DIRICHLET0 && c->co.bc != WRMG_BC_LID)
    throw Err{WRMG_E_UNSUPPORTED, "Navier-Stokes: bc must be WRMG_BC_DIRICHLET0 or WRMG_BC_LID"};
  c->ns = true;
  c->use_kron = false;
  THElement E;
  build_th_element(c->k, &E);
  c->th_nu = E.nu;
  c->th_np = E.np;
  {
    const int nu = E.nu, np = E.np;
    std::vector<double> ref(2 * nu * nu + 2 * nu * np), th(2 * nu * nu * nu);
    std::memcpy(ref.data(), E.Mh, nu * nu * sizeof(double));
    std::memcpy(ref.data() + nu * nu, E.Kh, nu * nu * sizeof(double));
    std::memcpy(ref.data() + 2 * nu * nu, E.Gh, 2 * nu * np * sizeof(double));
    std::memcpy(th.data(), E.Th, th.size() * sizeof(double));
    c->th_ref = dupload(ref, s);
    c->th_T = dupload(th, s);
  }
  std::vector<int> nys;
  std::vector<int> nxs = level_sizes(c->mesh.gnx, c->mesh.gny, c->mesh.ncoarse, &nys);
  // strips: the coarsest level -- the pinned-pressure direct
  // solve -- and every level narrower than 2 cells per strip run replicated on every
  // rank as a single-rank hierarchy (c->sub) below the partitioned levels
  c->strip = c->co.nranks > 1;
  if (c->strip) {
    int lrep = 1;
    for (int l = 0; l < (int)nxs.size(); ++l) {
      const int f = c->mesh.gnx / nxs[l];
      if (c->mesh.nx % f || c->mesh.nx / f < 2) lrep = std::max(lrep, l + 1);
    }
    if (lrep >= (int)nxs.size())
      throw Err{WRMG_E_UNSUPPORTED, "strips: the finest level's strip is narrower than 2 cells"};
    wrmg_mesh sm{};
    sm.gnx = nxs[lrep - 1];
    sm.gny = nys[lrep - 1];
    sm.x0 = 0;
    sm.nx = sm.gnx;
    sm.h = c->mesh.h * (double)(c->mesh.gnx / nxs[lrep - 1]);
    sm.ncoarse = c->mesh.ncoarse;
    wrmg_coeffs sc = c->co;
    sc.rank = 0;
    sc.nranks = 1;
    sc.loopback_hub = nullptr;
    sc.nccl_unique_id = nullptr;
    const wrmg_status st = wrmg_setup(&sm, c->k, c->q, c->N, c->dt, &sc, &c->sub);
    if (st != WRMG_OK) throw Err{st, std::string("replicated coarse hierarchy: ") + wrmg_last_error(nullptr, 0, 0, 0)};
    if ((int)c->sub->lv.size() != lrep) throw Err{WRMG_E_INVALID, "replicated coarse hierarchy: level count"};
    nxs.erase(nxs.begin(), nxs.begin() + lrep);
    nys.erase(nys.begin(), nys.begin() + lrep);
    make_strip_comm(c);
  } else if (c->mesh.x0 != 0 || c->mesh.nx != c->mesh.gnx) {
    throw Err{WRMG_E_INVALID, "a partial strip needs nranks > 1"};
  }
  const int nl = (int)nxs.size();
  std::vector<NSPlan> plans(nl);
  c->lv.resize(nl);
  for (int l = 0; l < nl; ++l) {
    const double h = c->mesh.h * (double)(c->mesh.gnx / nxs[l]);
    Level &L = c->lv[l];
    if (c->strip) {
      const int f = c->mesh.gnx / nxs[l];
      try {
        plan_ns_strip_level(nxs[l], nys[l], c->mesh.x0 / f, c->mesh.nx / f, h, c->k, c->co.bc, c->co.lid_speed,
                            c->co.rank, c->co.nranks, &plans[l], &L.st, &L.stp);
      } catch (const std::exception &e) {
        throw Err{WRMG_E_INVALID, e.what()};
      }
    } else {
      plan_ns_level(nxs[l], nys[l], h, c->k, c->co.bc, c->co.lid_speed, &plans[l]);
    }
    NSPlan &P = plans[l];
    L.nx = P.nx;
    L.ny = P.ny;
    L.h = h;
    L.Lx = P.Lux;
    L.Ly = P.Luy;
    L.Lux = P.Lux;
    L.Lpx = P.Lpx;
    L.Lu = P.Lu;
    L.Lp = P.Lp;
    L.nnode = P.ns;
    L.nfree = P.nfree;
    L.A.nrow = P.ns;
    L.A.nnz = (int64_t)P.col.size();
    L.A.rowptr = dupload(P.rowptr, s);
    L.A.col = dupload(P.col, s);
    L.A.val = dalloc<double>(P.col.size());
    L.A.val2 = dalloc<double>(P.col.size());
    L.h_con = P.con;
    L.con = dupload(P.con, s);
    L.vvptr = dupload(P.vvptr, s);
    L.nvv = P.vvptr.back();
    L.conv = dalloc<double>((size_t)L.nvv * c->nt);
    L.npatch = P.npatch;
    L.mp = P.mp;
    L.pnodes = dupload(P.pnodes, s);
    std::vector<double> w(P.ns, 0.0);
    for (int64_t i = 0; i < P.ns; ++i)
      if (P.mu[i] > 0) w[i] = (c->co.weights == WRMG_W_NONE) ? 1.0 : 1.0 / P.mu[i];
    L.wnode = dupload(w, s);
    double fl = 0.0;  // per (patch, slab): 2 m^2 (stored-inverse matvec) + 2 m_p^2 (jump)
    for (int32_t ps : P.psize) fl += 2.0 * ((double)c->nq * ps) * ((double)c->nq * ps) + 2.0 * (double)ps * ps;
    c->sweep_flops.push_back(fl * c->N);
    const int64_t m = (int64_t)c->nq * L.mp;
    if (m > 256 || ns_factor_smem((int)m, L.mp) > 227 * 1024)
      throw Err{WRMG_E_UNSUPPORTED, "Vanka patch system of size " + std::to_string(m) +
                                        " exceeds one CTA (shared-memory block inverse): lower q or degree"};
    L.mstride = (m * m + 1) & ~(int64_t)1;
    L.gLp = (int64_t)(c->k * nxs[l] + 1) * (c->k * nys[l] + 1);
    if (!c->strip) {  // single rank: the whole lattices
      L.st = StripInfo{};
      L.st.gnx = L.st.nx = L.st.nxl = nxs[l];
      L.st.own1 = L.Lux - 1;
      L.stp = L.st;
      L.stp.own1 = L.Lpx - 1;
      L.nfree_owned = L.nfree;
    } else {
      int64_t nfo = 0;
      for (int J = 0; J < P.Luy; ++J)
        for (int I = L.st.own0; I <= L.st.own1; ++I)
          nfo += !P.con[(int64_t)J * P.Lux + I] + !P.con[P.Lu + (int64_t)J * P.Lux + I];
      nfo += (int64_t)P.Lpy * (L.stp.own1 - L.stp.own0 + 1);
      L.nfree_owned = nfo;
      for (int b = 0; b < 4; ++b) L.hx[b] = dalloc<double>(halo_doubles(c, L));
    }
    if (l >= 1 || nl == 1 || c->strip) {  // the stored inverses are allocated after the slab windows are set
      L.nsinfo = dalloc<int32_t>((size_t)L.npatch * c->N);
      L.ppos = dalloc<int32_t>((size_t)L.npatch * L.mp * L.mp);
      L.pvv = dalloc<int32_t>((size_t)L.npatch * L.mp * L.mp);
    }
    if (l < nl - 1) {
      L.vr = dzalloc<double>(L.nnode * c->nt);
      L.vz = dzalloc<double>(L.nnode * c->nt);
      L.vt = dzalloc<double>(L.nnode * c->nt);
    }
    if (l < nl - 1 || c->strip) L.state = dzalloc<double>(L.nnode * c->nt);
    CK(cudaStreamSynchronize(s));
  }
  for (int l = 1; l < nl; ++l) {
    std::vector<int32_t> rp, ci, trp, tci;
    std::vector<double> v, tv;
    if (c->strip)
      plan_ns_strip_interpolation(plans[l - 1], c->lv[l - 1].st, c->lv[l - 1].stp, plans[l], c->lv[l].st,
                                  c->lv[l].stp, nys[l], rp, ci, v);
    else
      plan_ns_interpolation(plans[l - 1], plans[l], rp, ci, v);
    transpose_csr(plans[l].ns, plans[l - 1].ns, rp, ci, v, trp, tci, tv);
    Level &C = c->lv[l - 1];
    C.P.nrow = plans[l].ns;
    C.P.nnz = (int64_t)ci.size();
    C.P.rowptr = dupload(rp, s);
    C.P.col = dupload(ci, s);
    C.P.val = dupload(v, s);
    C.R.nrow = plans[l - 1].ns;
    C.R.nnz = (int64_t)tci.size();
    C.R.rowptr = dupload(trp, s);
    C.R.col = dupload(tci, s);
    C.R.val = dupload(tv, s);
    CK(cudaStreamSynchronize(s));
  }
  if (c->strip) {  // hand-over between level 0 (owned rows) and the replicated hierarchy (global sids)
    const Level &T = c->sub->lv.back();
    NSPlan gc;
    plan_ns_level(T.nx, T.ny, T.h, c->k, c->co.bc, c->co.lid_speed, &gc);
    StripInfo wu{}, wp{};
    wu.gnx = wu.nx = wu.nxl = T.nx;
    wp = wu;
    std::vector<int32_t> rp, ci, trp, tci;
    std::vector<double> v, tv;
    plan_ns_strip_interpolation(gc, wu, wp, plans[0], c->lv[0].st, c->lv[0].stp, nys[0], rp, ci, v);
    transpose_csr(plans[0].ns, gc.ns, rp, ci, v, trp, tci, tv);
    Level &X = c->xfer;
    X.P.nrow = plans[0].ns;
    X.P.nnz = (int64_t)ci.size();
    X.P.rowptr = dupload(rp, s);
    X.P.col = dupload(ci, s);
    X.P.val = dupload(v, s);
    X.R.nrow = gc.ns;
    X.R.nnz = (int64_t)tci.size();
    X.R.rowptr = dupload(trp, s);
    X.R.col = dupload(tci, s);
    X.R.val = dupload(tv, s);
    const int64_t ng = gc.ns * c->nt;
    c->sub_r = dzalloc<double>(ng);
    c->sub_z = dzalloc<double>(ng);
    c->sub_part = dzalloc<double>(ng);
    c->sub_w = dzalloc<double>(ng);
    c->sub_all = dzalloc<double>(ng * c->co.nranks);
    // state refresh: the largest owned-column block of any rank (rank 0 owns one more column)
    const Level &F = c->lv.back();
    const int ku = c->k + 1, kp = c->k;
    c->rf_chunk = ((int64_t)2 * F.Ly * (ku * F.st.nx + 1) + (int64_t)(F.Lp / F.Lpx) * (kp * F.stp.nx + 1)) * c->nt;
    c->rf_send = dzalloc<double>(c->rf_chunk);
    c->rf_recv = dzalloc<double>(c->rf_chunk * c->co.nranks);
    c->pj_sums = dzalloc<double>(c->nt);
    c->pj_all = dzalloc<double>(c->nt * c->co.nranks);
    CK(cudaStreamSynchronize(s));
  } else {
    Coarse &C = c->coarse;
    const NSPlan &P = plans[0];
    std::vector<int32_t> nodes;
    for (int64_t i = 0; i < P.ns; ++i)
      if (!P.con[i]) {
        if (i == 2 * P.Lu) C.pin = (int)nodes.size();  // first pressure DoF (R19)
        nodes.push_back((int32_t)i);
      }
    C.nfree = (int64_t)nodes.size();
    C.mp = (int)nodes.size();
    C.m = c->nq * C.mp;
    C.nnzj = 0;
    for (int32_t sd : nodes) C.nnzj += P.rowptr[sd + 1] - P.rowptr[sd];
    // dense per-slab blocks (m^2 doubles each, twice) and the end-trace recurrence's
    // 4 mc doubles of shared memory bound the coarse level
    if (C.m > 8192 || 4 * (size_t)C.mp * sizeof(double) > 220 * 1024)
      throw Err{WRMG_E_UNSUPPORTED, "coarse slab block larger than 8192 (raise ncoarse depth)"};
    C.nodes = dupload(nodes, s);
    C.nsD = dalloc<double>((size_t)c->N * C.m * C.m);
    C.nsinvT = dalloc<double>((size_t)c->N * C.m * C.m);
    C.nspiv = dalloc<int32_t>((size_t)c->N * C.m);
    C.nsinfo = dalloc<int32_t>(c->N);
    C.xq = dalloc<double>(P.ns);
    std::vector<int32_t> s2c(P.ns, -1);
    for (size_t i = 0; i < nodes.size(); ++i) s2c[nodes[i]] = (int32_t)i;
    C.sid2c = dupload(s2c, s);
    C.nsH = dalloc<double>((size_t)c->N * C.mp * C.m);
    C.nsG = dalloc<double>((size_t)c->N * C.mp * C.mp);
    C.nsZ = dalloc<double>((size_t)c->N * C.m);
    C.nsY = dalloc<double>((size_t)c->N * C.mp);
  }
  c->tmp = dalloc<double>(c->lv.back().nnode * c->nt);
  c->red = dalloc<double>(64 + 64 * kDotBlocksMax);
  {
    const Level &F = c->lv.back();
    c->proj = dalloc<double>(std::max<int64_t>(ns_project_scratch(F.Lp, c->nt), (F.Lp / F.Lpx + 1) * c->nt));
  }
  c->bcg = dupload(plans[nl - 1].g, s);
  for (auto &L : c->lv) {
    launch_ns_assemble_linear(geom(c, L), L.A, c->th_ref, s);
    if (L.ppos) launch_ns_patch_pos(geom(c, L), L.A, L.vvptr, L.pnodes, L.npatch, L.mp, L.ppos, L.pvv, s);
    check_launch();
  }
  CK(cudaStreamSynchronize(s));
  c->cheb = c->co.smoother == WRMG_SMOOTH_CHEBYSHEV;
  if (c->cheb) {
    if (c->co.cheb_steps == 0) c->co.cheb_steps = 50;
    c->lam.assign(nl, 0.0);
    c->cd.assign(nl, nullptr);
    c->cbr.assign(nl, nullptr);
    for (int l = c->strip ? 0 : 1; l < nl; ++l) {
      c->cd[l] = dzalloc<double>(c->lv[l].nnode * c->nt);
      c->cbr[l] = dzalloc<double>(c->lv[l].nnode * c->nt);
    }
  }
  ns_slab_windows(c);
  factor_all_ns(c, nullptr);
}

// r = b - F(u) on the finest level (eq. nsfem): the residual
// kernel with conv = R O(u) (Picard form of the convection, no Newton term).
void ns_nonlinear_residual(wrmg_ctx *c, const double *u, const double *b, double *r) {
  Level &L = c->lv.back();
  if (!c->conv_nl) c->conv_nl = dalloc<double>((size_t)L.nvv * c->nt);
  launch_ns_assemble_conv(geom(c, L), c->nt, c->co.reynolds, false, L.A, L.vvptr, u, c->conv_nl, c->th_T, c->stream);
  prof_residual(c, (int)c->lv.size() - 1, u, b, r, false, c->conv_nl);
}

int64_t ndof_level(const wrmg_ctx *c, int l) { return c->lv[l].nnode * c->nt; }

// z = B r on level l (H12): V(nu_pre, nu_post), zero initial guess.
// ------------------------------------------------------------ Chebyshev
void prof_sweep(wrmg_ctx *c, int l, const double *r, double *u, double om);

// lam_l: `steps` Arnoldi steps (CGS2) on B A from the seeded start vector, B one
// undamped sweep from zero; the estimate is the largest |Ritz value| (PAPER.md:366-371:
// "estimate the largest eigenvalue"; DESIGN.md R-cheb).
void reduce_to_host(wrmg_ctx *c, const double *dev, int nv, double *host);

double estimate_lambda(wrmg_ctx *c, int l) {
  cudaStream_t s = c->stream;
  Level &L = c->lv[l];
  const int64_t n = L.nnode * c->nt;
  const int steps = c->co.cheb_steps;
  std::vector<double *> V(steps + 1);
  for (auto &v : V) v = dzalloc<double>(n);
  double *w = dzalloc<double>(n), *t = dzalloc<double>(n);
  // strips: the Krylov vectors keep zero ghost columns, so the dots count owned rows;
  // every rank sums the all-gathered partial dots in rank order (reduce_to_host)
  auto dot = [&](const double *a, const double *b) {
    const int nb = multidot_blocks(n);
    const double *Vp[1] = {a};
    launch_multidot(Vp, 1, b, n, c->red + 64, nb, s);
    launch_reduce_partials(c->red + 64, nb, 1, c->red, s);
    double out = 0;
    reduce_to_host(c, c->red, 1, &out);
    return out;
  };
  // h = V[0..nv)^T w in chunks of 32 vectors
  auto multidot = [&](int nv, std::vector<double> &h) {
    h.assign(nv, 0.0);
    for (int c0 = 0; c0 < nv; c0 += 32) {
      const int k2 = std::min(32, nv - c0);
      const int nb = multidot_blocks(n);
      launch_multidot(V.data() + c0, k2, w, n, c->red + 64, nb, s);
      launch_reduce_partials(c->red + 64, nb, k2, c->red, s);
      reduce_to_host(c, c->red, k2, h.data() + c0);
    }
  };
  auto subtract = [&](int nv, const std::vector<double> &h) {  // w -= V h
    for (int c0 = 0; c0 < nv; c0 += 32) {
      const int k2 = std::min(32, nv - c0);
      CK(cudaMemcpyAsync(c->red, h.data() + c0, k2 * sizeof(double), cudaMemcpyHostToDevice, s));
      launch_multiaxpy(w, V.data() + c0, c->red, k2, n, -1.0, s);
    }
  };
  if (!c->strip) {
    launch_fill_uniform(V[0], n, 0, c->co.cheb_seed, s);
  } else {  // R6 generator at the global canonical ids: local row J holds global columns G0 ..
    FieldView f[3];
    const int nf = level_fields(c, L, f);
    for (int i = 0; i < nf; ++i) {
      const int64_t GLx = (int64_t)f[i].k * f[i].S->gnx + 1, rowlen = (int64_t)f[i].Lx * c->nt;
      for (int J = 0; J < f[i].Ly; ++J)
        launch_fill_uniform(V[0] + f[i].off + J * rowlen, rowlen,
                            (uint64_t)((f[i].goff + J * GLx + f[i].S->G0) * c->nt), c->co.cheb_seed, s);
    }
    zero_ghosts(c, L, V[0]);
  }
  launch_ns_mask(L.nnode, c->nt, L.con, nullptr, V[0], V[0], s);  // constrained rows 0
  launch_scale(V[0], V[0], 1.0 / std::sqrt(dot(V[0], V[0])), n, s);
  std::vector<double> H((size_t)(steps + 1) * steps, 0.0), h, h2;
  for (int j = 0; j < steps; ++j) {
    if (c->strip) halo_forward(c, L, V[j]);
    prof_residual(c, l, V[j], nullptr, t, false);  // t = A v_j
    CK(cudaMemsetAsync(w, 0, n * sizeof(double), s));
    if (c->strip) {
      zero_ghosts(c, L, V[j]);
      halo_forward(c, L, t);
      sweep_strip(c, l, t, w, 1.0);                 // w = B A v_j
      zero_ghosts(c, L, w);
    } else {
      prof_sweep(c, l, t, w, 1.0);                  // w = B A v_j
    }
    multidot(j + 1, h);
    subtract(j + 1, h);
    multidot(j + 1, h2);
    subtract(j + 1, h2);
    const double hn = std::sqrt(dot(w, w));
    for (int i = 0; i <= j; ++i) H[(size_t)i * steps + j] = h[i] + h2[i];
    H[(size_t)(j + 1) * steps + j] = hn;
    if (hn <= 0.0) break;
    launch_scale(V[j + 1], w, 1.0 / hn, n, s);
  }
  CK(cudaStreamSynchronize(s));
  for (auto v : V) dfree(v);
  dfree(w);
  dfree(t);
  // largest |Ritz value|: eigenvalues of the square Hessenberg (R-cheb)
  std::vector<double> Hs(H.begin(), H.begin() + (size_t)steps * steps), wr, wi;
  if (!hessenberg_eigenvalues(Hs, steps, wr, wi)) throw Err{WRMG_E_NOT_CONVERGED, "Ritz values did not converge"};
  double mx = 0.0;
  for (int i = 0; i < steps; ++i) mx = std::max(mx, std::hypot(wr[i], wi[i]));
  return mx;
}

// nu Chebyshev steps for B A x = B b on [0.25 lam, 1.05 lam]:
// d_0 = B r_0 / theta, d_k = rho_k rho_{k-1} d_{k-1} + (2 rho_k / delta) B r_k, x += d_k.
void cheb_smooth(wrmg_ctx *c, int l, const double *b, double *u, bool u_zero, int nu) {
  cudaStream_t s = c->stream;
  Level &L = c->lv[l];
  const int64_t n = L.nnode * c->nt;
  double *t = (l == (int)c->lv.size() - 1) ? c->tmp : L.vt;
  double *d = c->cd[l], *br = c->cbr[l];
  const double lam = c->lam[l], lo = 0.25 * lam, hi = 1.05 * lam;
  const double theta = 0.5 * (hi + lo), delta = 0.5 * (hi - lo), sigma = theta / delta;
  double rho = 1.0 / sigma;
  for (int k2 = 0; k2 < nu; ++k2) {
    const double *res = b;
    if (k2 > 0 || !u_zero) {
      prof_residual(c, l, u, b, t, false);  // strips: u's ghosts are current (see below)
      res = t;
    }
    CK(cudaMemsetAsync(br, 0, n * sizeof(double), s));
    if (c->strip) {
      if (res != b) halo_forward(c, L, t);  // b's ghosts were refreshed by the caller
      sweep_strip(c, l, res, br, 1.0);      // br valid on owned and ghost columns
    } else {
      prof_sweep(c, l, res, br, 1.0);
    }
    double c1 = 0.0, c2 = 1.0 / theta;
    if (k2 > 0) {
      const double rn = 1.0 / (2.0 * sigma - rho);
      c1 = rn * rho;
      c2 = 2.0 * rn / delta;
      rho = rn;
    }
    launch_cheb_update(n, c1, c2, br, d, u, s);
  }
}

// V(nu_pre, nu_post) on a strip: r is valid on owned columns
// (ghosts refreshed here), z leaves valid on owned and ghost columns.
void vcycle_level(wrmg_ctx *c, int l, const double *r, double *z);

// Below the coarsest partitioned level: the restriction of the owned fine rows into
// the replicated level (partial sums), all-reduced in rank order; the replicated
// V-cycle (c->sub, identical on every rank); prolongation to the owned fine rows.
void sub_cycle(wrmg_ctx *c, const double *t, double *z) {
  cudaStream_t s = c->stream;
  wrmg_ctx *S = c->sub;
  const Level &T = S->lv.back();
  const int64_t ng = T.nnode * c->nt;
  {
    PScope ps(c, WRMG_K_RESTRICT, 0, 8.0 * (c->lv[0].nnode + T.nnode) * c->nt, 2.0 * c->xfer.R.nnz * c->nt);
    launch_restrict(c->xfer, c->nt, t, c->sub_part, s);
  }
  comm_call(c, [&] { c->comm->allgather(c->sub_part, c->sub_all, (size_t)ng, s); });
  launch_sum_chunks(c->sub_all, c->comm->nranks, ng, c->sub_r, s);
  if (c->ns) ns_project(S, T, c->sub_r);
  vcycle_level(S, (int)S->lv.size() - 1, c->sub_r, c->sub_z);
  {
    PScope ps(c, WRMG_K_PROLONG, 0, 8.0 * (2 * c->lv[0].nnode + T.nnode) * c->nt, 2.0 * c->xfer.P.nnz * c->nt);
    launch_prolong_add(c->xfer, c->nt, c->sub_z, z, s);
  }
}

void vcycle_strip(wrmg_ctx *c, int l, const double *r, double *z) {
  cudaStream_t s = c->stream;
  Level &L = c->lv[l];
  if (l == 0 && !c->sub) {
    coarse_strip(c, r, z);
    return;
  }
  const int64_t nd = L.nnode * c->nt;
  double *t = (l == (int)c->lv.size() - 1) ? c->tmp : L.vt;
  const double om = c->co.omega_mg;
  halo_forward(c, L, const_cast<double *>(r));
  CK(cudaMemsetAsync(z, 0, nd * sizeof(double), s));
  if (c->cheb) {
    cheb_smooth(c, l, r, z, true, c->co.nu_pre);
  } else {
    for (int it = 0; it < c->co.nu_pre; ++it) {
      if (it == 0) {
        sweep_strip(c, l, r, z, om);
      } else {
        prof_residual(c, l, z, r, t, false);
        halo_forward(c, L, t);
        sweep_strip(c, l, t, z, om);
      }
    }
  }
  prof_residual(c, l, z, r, t, c->co.nu_pre == 0);
  if (l == 0) {
    sub_cycle(c, t, z);
  } else {
    Level &C = c->lv[l - 1];
    {
      PScope ps(c, WRMG_K_RESTRICT, l, 8.0 * (L.nnode + C.nnode) * c->nt, 2.0 * C.R.nnz * c->nt);
      launch_restrict(C, c->nt, t, C.vr, s);  // R = P^T over owned fine rows
    }
    halo_reverse_add(c, C, C.vr);
    if (c->ns) ns_project(c, C, C.vr);
    vcycle_strip(c, l - 1, C.vr, C.vz);
    {
      PScope ps(c, WRMG_K_PROLONG, l, 8.0 * (2 * L.nnode + C.nnode) * c->nt, 2.0 * C.P.nnz * c->nt);
      launch_prolong_add(C, c->nt, C.vz, z, s);  // owned fine rows
    }
  }
  halo_forward(c, L, z);
  if (c->cheb) {
    cheb_smooth(c, l, r, z, false, c->co.nu_post);
  } else {
    for (int it = 0; it < c->co.nu_post; ++it) {
      prof_residual(c, l, z, r, t, false);
      halo_forward(c, L, t);
      sweep_strip(c, l, t, z, om);
    }
  }
  check_launch();
}

void vcycle_level(wrmg_ctx *c, int l, const double *r, double *z) {
  if (c->strip) {
    vcycle_strip(c, l, r, z);
    return;
  }
  cudaStream_t s = c->stream;
  Level &L = c->lv[l];
  if (l == 0 && c->ns) {
    const Coarse &C = c->coarse;
    PScope ps(c, WRMG_K_COARSE, 0, 8.0 * c->N * (double)C.m * C.m + 16.0 * L.nnode * c->nt,
              2.0 * c->N * (double)C.m * C.m);
    static const bool march = [] {  // WRMG_NS_COARSE_MARCH=1: the slab-by-slab cluster march (A/B)
      const char *e = getenv("WRMG_NS_COARSE_MARCH");
      return e && e[0] == '1';
    }();
    if (march)
      launch_ns_coarse_solve(c->q, c->N, C.mp, C.pin, C.nodes, L.A, C.nsinvT, r, z, C.xq, L.nnode, C.nnzj, s);
    else
      launch_ns_coarse_solve_pint(c->q, c->N, C.mp, C.pin, C.nodes, C.nsinvT, C.nsH, C.nsG, C.nsZ, C.nsY, r, z,
                                  L.nnode, s);
    ns_project(c, L, z);
    return;
  }
  if (l == 0) {
    const Coarse &C = c->coarse;
    PScope ps(c, WRMG_K_COARSE, 0, 16.0 * C.nfree * c->nt + 8.0 * L.nnode * c->nt,
              2.0 * c->N * ((double)C.m * C.m + (double)C.m * C.mp));
    if (c->coarse_kron)
      launch_coarse_solve_kron(C, L, c->q, c->N, r, z, s);
    else
      launch_coarse_solve(C, L, c->q, c->N, r, z, s);
    return;
  }
  const int64_t nd = ndof_level(c, l);
  double *t = (l == (int)c->lv.size() - 1) ? c->tmp : L.vt;
  const double om = c->co.omega_mg;
  CK(cudaMemsetAsync(z, 0, nd * sizeof(double), s));
  if (c->cheb) {
    cheb_smooth(c, l, r, z, true, c->co.nu_pre);
  } else {
    for (int it = 0; it < c->co.nu_pre; ++it) {
      if (it == 0) {
        prof_sweep(c, l, r, z, om);  // u = 0: residual is r itself
      } else {
        prof_residual(c, l, z, r, t, false);
        prof_sweep(c, l, t, z, om);
      }
    }
  }
  prof_residual(c, l, z, r, t, c->co.nu_pre == 0);
  Level &C = c->lv[l - 1];
  {
    PScope ps(c, WRMG_K_RESTRICT, l, 8.0 * (L.nnode + C.nnode) * c->nt, 2.0 * C.R.nnz * c->nt);
    launch_restrict(C, c->nt, t, C.vr, s);
  }
  if (c->ns) ns_project(c, C, C.vr);
  vcycle_level(c, l - 1, C.vr, C.vz);
  {
    PScope ps(c, WRMG_K_PROLONG, l, 8.0 * (2 * L.nnode + C.nnode) * c->nt, 2.0 * C.P.nnz * c->nt);
    launch_prolong_add(C, c->nt, C.vz, z, s);
  }
  if (c->cheb) {
    cheb_smooth(c, l, r, z, false, c->co.nu_post);
  } else {
    for (int it = 0; it < c->co.nu_post; ++it) {
      prof_residual(c, l, z, r, t, false);
      prof_sweep(c, l, t, z, om);
    }
  }
  check_launch();
}

// Small transfers of the Krylov loop through mapped pinned memory and a copy
// kernel on the context's stream: they never queue behind bulk copies that other
// streams (e.g. a serving loop's next input) keep on the copy engines.
double *hmap(wrmg_ctx *c) {
  if (!c->hmap) {
    const int P = c->comm ? c->comm->nranks : 1;
    c->hmap_cap = std::max(1024, 64 * P);
    CK(cudaHostAlloc((void **)&c->hmap, 2 * (size_t)c->hmap_cap * sizeof(double), cudaHostAllocMapped));
  }
  return c->hmap;
}
void small_d2h(wrmg_ctx *c, const double *dev, double *host, int nv) {  // synchronises
  double *hm = hmap(c);
  if (nv > c->hmap_cap) throw Err{WRMG_E_INVALID, "small_d2h: transfer larger than the mapped buffer"};
  launch_scale(hm, dev, 1.0, nv, c->stream);
  CK(cudaStreamSynchronize(c->stream));
  std::memcpy(host, hm, nv * sizeof(double));
}
void small_h2d(wrmg_ctx *c, const double *host, double *dev, int nv) {  // caller synchronises before reuse
  double *hm = hmap(c) + c->hmap_cap;
  if (nv > c->hmap_cap) throw Err{WRMG_E_INVALID, "small_h2d: transfer larger than the mapped buffer"};
  std::memcpy(hm, host, nv * sizeof(double));
  launch_scale(dev, hm, 1.0, nv, c->stream);
}

// Host copy of nv reduction results at dev (<= 64).  Strips: every rank's values
// are all-gathered and summed in rank order, so all ranks hold bitwise-identical
// global sums (and take identical host-side decisions).
void reduce_to_host(wrmg_ctx *c, const double *dev, int nv, double *host) {
  cudaStream_t s = c->stream;
  if (!c->strip || c->comm->nranks == 1) {
    small_d2h(c, dev, host, nv);
    return;
  }
  const int P = c->comm->nranks;
  if (!c->gred) c->gred = dalloc<double>((size_t)P * 64);
  comm_call(c, [&] { c->comm->allgather(dev, c->gred, (size_t)nv, s); });
  std::vector<double> all((size_t)P * nv);
  small_d2h(c, c->gred, all.data(), (int)all.size());
  for (int i = 0; i < nv; ++i) {
    double t = 0.0;
    for (int q = 0; q < P; ++q) t += all[(size_t)q * nv + i];
    host[i] = t;
  }
}

// Global dot product (owned rows: strips pass vectors with zeroed ghost columns).
double dot_host(wrmg_ctx *c, const double *a, const double *b, int64_t n) {
  PScope ps(c, WRMG_K_KRYLOV, (int)c->lv.size() - 1, 16.0 * n, 2.0 * n);
  int nb = multidot_blocks(n);
  const double *V[1] = {a};
  launch_multidot(V, 1, b, n, c->red + 64, nb, c->stream);
  launch_reduce_partials(c->red + 64, nb, 1, c->red, c->stream);
  double out = 0;
  reduce_to_host(c, c->red, 1, &out);
  return out;
}

// Every exported entry point runs on the context's device and restores the
// caller's current device on return (wrmg_setup used to leave the
// calling thread on coeffs.device and later calls used whatever was current).
// Entry-point guard: the context's device for the call (the caller's restored after), and
// an NVTX range named after the entry point.
struct DevGuard {
  int prev = -1, dev = -1;
  bool named = false;
  explicit DevGuard(int d, const char *name = nullptr) : dev(d) {
    if (name) {
      nvtxRangePushA(name);
      named = true;
    }
    if (dev < 0 || cudaGetDevice(&prev) != cudaSuccess) {
      dev = -1;
      return;
    }
    if (prev != dev) cudaSetDevice(dev);
  }
  explicit DevGuard(const wrmg_ctx *c, const char *name = nullptr) : DevGuard(c ? c->co.device : -1, name) {}
  ~DevGuard() {
    if (dev >= 0 && prev != dev) cudaSetDevice(prev);
    if (named) nvtxRangePop();
  }
};

}  // namespace

// Device vectors must be 16-byte aligned (the kernels move 16-byte pairs and TMA boxes;
// cudaMalloc and torch allocations are): a view at an odd double offset is rejected.
static bool al16(const void *p) { return ((uintptr_t)p & 15u) == 0; }
template <class... T>
static bool al16(const void *p, T... rest) {
  return al16(p) && al16(rest...);
}

extern "C" {

wrmg_status wrmg_plan(const wrmg_mesh *mesh, int32_t degree, int32_t q, int32_t nslabs, wrmg_layout_t *out) {
  try {
    validate(mesh, degree, q, nslabs, 1.0);
    if (!out) throw Err{WRMG_E_INVALID, "out is NULL"};
    std::vector<int> nys;
    int nc = mesh->ncoarse > 0 ? mesh->ncoarse : 4;
    std::vector<int> nxs = level_sizes(mesh->gnx, mesh->gny, nc, &nys);
    PlanLevel P;
    plan_level(mesh->gnx, mesh->gny, mesh->h, degree, &P);
    std::memset(out, 0, sizeof(*out));
    out->nnode = P.nnode;
    out->nt = (int64_t)nslabs * (q + 1);
    out->ndof = P.nnode * out->nt;
    out->nfree_st = P.nfree * out->nt;
    out->lx = P.Lx;
    out->ly = P.Ly;
    out->nlevels = (int)nxs.size();
    out->degree = degree;
    out->q = q;
    out->nslabs = nslabs;
    out->npatch = P.npatch;
    int mx = 0;
    for (int32_t s : P.psize) mx = std::max(mx, (int)s);
    out->mp_max = mx;
    out->npatch_types = P.ntypes;
    return WRMG_OK;
  } catch (const Err &e) {
    return fail(nullptr, e);
  }
}

wrmg_status wrmg_plan_patches(const wrmg_mesh *mesh, int32_t degree, int32_t *nodes, int32_t *sizes) {
  try {
    validate(mesh, degree, 0, 1, 1.0);
    PlanLevel P;
    plan_level(mesh->gnx, mesh->gny, mesh->h, degree, &P);
    int mx = 0;
    for (int32_t s : P.psize) mx = std::max(mx, (int)s);
    if (nodes)
      for (int64_t p = 0; p < P.npatch; ++p)
        for (int j = 0; j < mx; ++j) nodes[p * mx + j] = j < P.psize[p] ? P.pnodes[p * P.mp + j] : -1;
    if (sizes)
      for (int64_t p = 0; p < P.npatch; ++p) sizes[p] = P.psize[p];
    return WRMG_OK;
  } catch (const Err &e) {
    return fail(nullptr, e);
  }
}

wrmg_status wrmg_plan_strip(const wrmg_mesh *mesh, int32_t degree, int32_t rank, int32_t nranks, int32_t *info,
                            int32_t *patch_vertex, int64_t *npatch) {
  try {
    validate(mesh, degree, 0, 1, 1.0);
    if (!info || nranks < 1 || rank < 0 || rank >= nranks) throw Err{WRMG_E_INVALID, "bad strip query"};
    PlanLevel P;
    StripInfo S;
    plan_strip_level(mesh->gnx, mesh->gny, mesh->x0, mesh->nx, mesh->h, degree, rank, nranks, &P, &S);
    const int32_t v[16] = {S.G0, S.own0, S.own1, S.lg0, S.nlg, S.rg0, S.nrg, S.sl0, S.nsl, S.sr0, S.nsr, P.Lx, P.Ly,
                           S.cx0, S.nxl, 0};
    std::memcpy(info, v, sizeof(v));
    if (npatch) *npatch = P.npatch;
    if (patch_vertex)  // global vertex ids J (gnx + 1) + I
      for (int64_t p = 0; p < P.npatch; ++p) {
        const int vi = P.pvert[p] % (S.nxl + 1) + S.cx0, vj = P.pvert[p] / (S.nxl + 1);
        patch_vertex[p] = vj * (mesh->gnx + 1) + vi;
      }
    return WRMG_OK;
  } catch (const Err &e) {
    return fail(nullptr, e);
  }
}

wrmg_status wrmg_plan_ns_strip(const wrmg_mesh *mesh, int32_t degree, int32_t rank, int32_t nranks, int32_t *info,
                               int32_t *patch_vertex, int32_t *patch_sids, int64_t *npatch, int32_t *mp) {
  try {
    validate(mesh, degree + 1, 0, 1, 1.0);
    if (!info || nranks < 1 || rank < 0 || rank >= nranks || degree < 1 || degree > 2)
      throw Err{WRMG_E_INVALID, "bad strip query"};
    NSPlan P;
    StripInfo Su, Sp;
    try {
      plan_ns_strip_level(mesh->gnx, mesh->gny, mesh->x0, mesh->nx, mesh->h, degree, WRMG_BC_LID, 1.0, rank, nranks,
                          &P, &Su, &Sp);
    } catch (const std::exception &e) {
      throw Err{WRMG_E_INVALID, e.what()};
    }
    const int Lpy = P.Lpy;
    const int32_t v[32] = {Su.G0, Su.own0, Su.own1, Su.lg0, Su.nlg, Su.rg0, Su.nrg, Su.sl0, Su.nsl, Su.sr0, Su.nsr,
                           P.Lux, P.Luy, Su.cx0, Su.nxl, 0,
                           Sp.G0, Sp.own0, Sp.own1, Sp.lg0, Sp.nlg, Sp.rg0, Sp.nrg, Sp.sl0, Sp.nsl, Sp.sr0, Sp.nsr,
                           P.Lpx, Lpy, Sp.cx0, Sp.nxl, 0};
    std::memcpy(info, v, sizeof(v));
    if (npatch) *npatch = P.npatch;
    if (mp) *mp = P.mp;
    const int64_t GLux = (int64_t)(degree + 1) * mesh->gnx + 1, GLu = GLux * P.Luy, GLpx = (int64_t)degree * mesh->gnx + 1;
    for (int64_t p = 0; p < P.npatch; ++p) {
      if (patch_vertex) patch_vertex[p] = P.pvert[p];
      if (patch_sids)
        for (int e = 0; e < P.mp; ++e) {
          const int32_t l = P.pnodes[p * P.mp + e];
          int64_t g = -1;
          if (l >= 0 && l < 2 * P.Lu) {
            const int64_t d = l / P.Lu, i = l - d * P.Lu;
            g = d * GLu + (i / P.Lux) * GLux + (i % P.Lux) + Su.G0;
          } else if (l >= 0) {
            const int64_t j = l - 2 * P.Lu;
            g = 2 * GLu + (j / P.Lpx) * GLpx + (j % P.Lpx) + Sp.G0;
          }
          patch_sids[p * P.mp + e] = (int32_t)g;
        }
    }
    return WRMG_OK;
  } catch (const Err &e) {
    return fail(nullptr, e);
  }
}

wrmg_status wrmg_setup(const wrmg_mesh *mesh, int32_t degree, int32_t q, int32_t nslabs, double dt,
                       const wrmg_coeffs *coeffs, wrmg_ctx **out) {
  wrmg_ctx *c = nullptr;
  DevGuard dg_(coeffs ? coeffs->device : -1, "wrmg_setup");
  try {
    if (!out) throw Err{WRMG_E_INVALID, "out is NULL"};
    *out = nullptr;
    validate(mesh, degree, q, nslabs, dt);
    if (!coeffs) throw Err{WRMG_E_INVALID, "coeffs is NULL"};
    if (coeffs->problem != WRMG_HEAT && coeffs->problem != WRMG_NAVIER_STOKES)
      throw Err{WRMG_E_UNSUPPORTED, "problem must be WRMG_HEAT or WRMG_NAVIER_STOKES"};
    if (coeffs->problem == WRMG_HEAT && coeffs->bc != WRMG_BC_DIRICHLET0 && coeffs->bc != WRMG_BC_NEUMANN)
      throw Err{WRMG_E_UNSUPPORTED, "heat: bc must be WRMG_BC_DIRICHLET0 or WRMG_BC_NEUMANN"};
    if (coeffs->smoother == WRMG_SMOOTH_CHEBYSHEV && (coeffs->cheb_steps < 0 || coeffs->cheb_steps > 63))
      throw Err{WRMG_E_UNSUPPORTED, "Chebyshev smoothing: cheb_steps <= 63"};
    if (coeffs->problem == WRMG_HEAT && !(coeffs->kappa > 0)) throw Err{WRMG_E_INVALID, "kappa must be > 0"};
    if (coeffs->orth != WRMG_ORTH_CGS && coeffs->orth != WRMG_ORTH_CGS2)
      throw Err{WRMG_E_INVALID, "orth must be WRMG_ORTH_CGS or WRMG_ORTH_CGS2"};
    c = new wrmg_ctx();
    c->mesh = *mesh;
    if (c->mesh.nx == 0) c->mesh.nx = mesh->gnx;
    if (c->mesh.ncoarse <= 0) c->mesh.ncoarse = 4;
    c->co = *coeffs;
    // factor_mode 0 (AUTO): Kronecker-diagonalised patch solves for the heat operator
    // (N <= 256); 1 (LU): per-class LU factors and the split-form sweep
    c->use_kron = coeffs->factor_mode == 0 && nslabs <= 256;
    if (!(c->co.omega_mg > 0)) c->co.omega_mg = 1.0;
    if (c->co.nu_pre <= 0 && c->co.nu_post <= 0) c->co.nu_pre = c->co.nu_post = 1;
    c->k = degree;
    c->q = q;
    c->nq = q + 1;
    c->N = nslabs;
    c->nt = (int64_t)nslabs * c->nq;
    c->dt = dt;
    CK(cudaSetDevice(coeffs->device));
    c->stream = (cudaStream_t)coeffs->stream;
    cudaStream_t s = c->stream;
    build_ref_element(degree, &c->ref);
    build_temporal(q, dt, &c->tm);
    for (int a = 0; a < c->nq; ++a)
      for (int b = 0; b < c->nq; ++b) {
        double want = (a == 0 && b == q) ? 1.0 : 0.0;
        if (std::fabs(c->tm.E1[a * c->nq + b] - want) > 1e-14)
          throw Err{WRMG_E_UNSUPPORTED, "E1 is not e_0 e_q^T (R2 temporal basis)"};
      }
    {
      int nloc = c->ref.nloc;
      std::vector<double> ref(2 * nloc * nloc);
      std::memcpy(ref.data(), c->ref.M, nloc * nloc * sizeof(double));
      std::memcpy(ref.data() + nloc * nloc, c->ref.K, nloc * nloc * sizeof(double));
      c->ref_dev = dupload(ref, s);
    }
    if (coeffs->problem == WRMG_NAVIER_STOKES) {
      setup_ns(c);
      *out = c;
      return WRMG_OK;
    }
    std::vector<int> nys;
    std::vector<int> nxs = level_sizes(mesh->gnx, mesh->gny, c->mesh.ncoarse, &nys);
    c->strip = coeffs->nranks > 1;
    const bool neumann = coeffs->bc == WRMG_BC_NEUMANN;
    // strips: levels whose strip is narrower than 2 cells are agglomerated -- they run
    // replicated on every rank as a complete single-rank hierarchy (c->sub) below the
    // coarsest partitioned level
    int lrep = 0;
    if (c->strip)
      for (int l = 0; l < (int)nxs.size(); ++l) {
        const int f = mesh->gnx / nxs[l];
        if (c->mesh.nx % f || c->mesh.nx / f < 2) lrep = l + 1;
      }
    if (lrep >= (int)nxs.size())
      throw Err{WRMG_E_UNSUPPORTED, "strips: the finest level's strip is narrower than 2 cells"};
    if (lrep > 0) {
      wrmg_mesh sm{};
      sm.gnx = nxs[lrep - 1];
      sm.gny = nys[lrep - 1];
      sm.x0 = 0;
      sm.nx = sm.gnx;
      sm.h = mesh->h * (double)(mesh->gnx / nxs[lrep - 1]);
      sm.ncoarse = c->mesh.ncoarse;
      wrmg_coeffs sc = *coeffs;
      sc.rank = 0;
      sc.nranks = 1;
      sc.loopback_hub = nullptr;
      sc.nccl_unique_id = nullptr;
      const wrmg_status st = wrmg_setup(&sm, degree, q, nslabs, dt, &sc, &c->sub);
      if (st != WRMG_OK) throw Err{st, std::string("replicated coarse hierarchy: ") + wrmg_last_error(nullptr, 0, 0, 0)};
      nxs.erase(nxs.begin(), nxs.begin() + lrep);
      nys.erase(nys.begin(), nys.begin() + lrep);
    }
    const int nl = (int)nxs.size();
    std::vector<PlanLevel> plans(nl);
    c->lv.resize(nl);
    if (c->strip) {
      make_strip_comm(c);
    } else if (c->mesh.x0 != 0 || c->mesh.nx != mesh->gnx) {
      throw Err{WRMG_E_INVALID, "a partial strip needs nranks > 1"};
    }
    for (int l = 0; l < nl; ++l) {
      double h = mesh->h * (double)(mesh->gnx / nxs[l]);
      Level &L = c->lv[l];
      if (c->strip) {
        const int f = mesh->gnx / nxs[l];
        plan_strip_level(nxs[l], nys[l], c->mesh.x0 / f, c->mesh.nx / f, h, degree, coeffs->rank, coeffs->nranks,
                         &plans[l], &L.st, neumann);
      } else {
        plan_level(nxs[l], nys[l], h, degree, &plans[l], neumann);
        L.st = StripInfo{};
        L.st.gnx = nxs[l];
        L.st.nx = nxs[l];
        L.st.nxl = nxs[l];
        L.st.own1 = degree * nxs[l];
      }
      PlanLevel &P = plans[l];
      {
        int64_t nfo = 0;
        for (int J = 0; J < P.Ly; ++J)
          for (int I = L.st.own0; I <= L.st.own1; ++I) nfo += !P.con[(int64_t)J * P.Lx + I];
        L.nfree_owned = nfo;
      }
      L.nx = P.nx;
      L.ny = P.ny;
      L.h = h;
      L.Lx = P.Lx;
      L.Ly = P.Ly;
      L.nnode = P.nnode;
      L.nfree = P.nfree;
      L.A.nrow = P.nnode;
      L.A.nnz = (int64_t)P.col.size();
      L.A.rowptr = dupload(P.rowptr, s);
      L.A.col = dupload(P.col, s);
      L.A.val = dalloc<double>(P.col.size());
      L.A.val2 = dalloc<double>(P.col.size());
      L.h_con = P.con;
      L.con = dupload(P.con, s);
      L.npatch = P.npatch;
      L.mp = P.mp;
      L.ntypes = P.ntypes;
      L.pnodes = dupload(P.pnodes, s);
      L.ptype = dupload(P.ptype, s);
      L.h_type_rep = P.type_rep;
      L.type_rep = dupload(P.type_rep, s);
      std::vector<double> w(P.nnode, 0.0);
      for (int64_t i = 0; i < P.nnode; ++i)
        if (P.mu[i] > 0) w[i] = (c->co.weights == WRMG_W_NONE) ? 1.0 : 1.0 / P.mu[i];
      L.wnode = dupload(w, s);
      int m = c->nq * L.mp;
      L.Dblk = dalloc<double>((size_t)L.ntypes * m * m);
      L.Dinv = dalloc<double>((size_t)L.ntypes * m * m);
      L.G = dalloc<double>((size_t)L.ntypes * m * L.mp);
      L.piv = dalloc<int32_t>((size_t)L.ntypes * m);
      L.info = dalloc<int32_t>(L.ntypes);
      L.rcls = dupload(P.rcls, s);
      L.h_rcls = P.rcls;
      L.h_cls_rep = P.cls_rep;
      if (c->use_kron && c->nq <= (degree == 3 ? 3 : 4) && degree >= 2 && P.npatch >= 1000 && !sym_disabled()) {
        // symmetry-reduced sweep for the interior vertex-star class (host_sym.cu): the most frequent class
        std::vector<int64_t> cnt(P.ntypes, 0);
        for (int64_t p = 0; p < P.npatch; ++p) ++cnt[P.ptype[p]];
        const int cls = (int)(std::max_element(cnt.begin(), cnt.end()) - cnt.begin());
        std::vector<int32_t> perm;
        int counts[3];
        if (plan_sym_class(P, degree, cls, perm, counts)) {
          std::vector<int32_t> sn;
          sn.reserve((size_t)cnt[cls] * perm.size());
          for (int64_t p = 0; p < P.npatch; ++p)
            if (P.ptype[p] == cls)
              for (int32_t sl : perm) sn.push_back(P.pnodes[p * P.mp + sl]);
          L.sym_ok = true;
          L.sym_cls = cls;
          L.nsym = cnt[cls];
          L.sym_nodes = dupload(sn, s);
          plan_sym_tiles(P, degree, cls, (int)perm.size(), sn, L, s);
          // CSR positions of the representative patch block (values read at factor time)
          const int64_t rep = P.type_rep[cls];
          const int mps = (int)perm.size();
          L.sym_pos.assign((size_t)mps * mps, -1);
          for (int a2 = 0; a2 < mps; ++a2) {
            const int32_t i = P.pnodes[rep * P.mp + perm[a2]];
            for (int b2 = 0; b2 < mps; ++b2) {
              const int32_t j = P.pnodes[rep * P.mp + perm[b2]];
              for (int32_t e = P.rowptr[i]; e < P.rowptr[i + 1]; ++e)
                if (P.col[e] == j) L.sym_pos[(size_t)a2 * mps + b2] = e;
            }
          }
        }
      }
      if (c->use_kron) {
        const int ld = (L.mp + 1) & ~1;
        L.kV = dalloc<double>((size_t)L.ntypes * L.mp * ld);
        L.kVT = dalloc<double>((size_t)L.ntypes * L.mp * ld);
        L.kS = dalloc<double>((size_t)L.ntypes * L.mp * c->nq * c->nq);
        L.ksig = dalloc<double>((size_t)L.ntypes * L.mp);
        const int C = (c->N + 31) / 32;
        // patches per CTA: 8 warps' worth, or 1 when that leaves fewer than 2 CTAs per SM
        // (coarse levels are latency-bound)
        int pp = std::max(1, 8 / C);
        const int ex = L.sym_ok ? L.sym_cls : -1;  // the symmetric class runs in kernels_sweep_sym.cu
        std::vector<int32_t> cp, ct;
        plan_sweep_ctas(P, pp, cp, ct, ex);
        if (pp > 1 && (int)ct.size() < 2 * num_sms()) {
          pp = 1;
          plan_sweep_ctas(P, pp, cp, ct, ex);
        }
        L.kron_pp = pp;
        L.kron_ncta = (int)ct.size();
        L.cta_patch = dupload(cp, s);
        L.cta_type = dupload(ct, s);
        plan_sweep_ctas(P, 1, cp, ct, ex);
        L.kron_ncta1 = (int)ct.size();
        L.cta_patch1 = dupload(cp, s);
        L.cta_type1 = dupload(ct, s);
        plan_sweep_ctas(P, 8, cp, ct, ex);
        L.kron_ngrp8 = (int)ct.size();
        L.grp_patch8 = dupload(cp, s);
        L.grp_type8 = dupload(ct, s);
        if (coeffs->scatter == WRMG_SCATTER_COLOUR) {  // per-colour work lists (deterministic scatter)
          std::vector<uint8_t> pc(P.npatch);
          for (int64_t p = 0; p < P.npatch; ++p) {
            const int vi = P.pvert[p] % (P.nx + 1) + L.st.cx0, vj = P.pvert[p] / (P.nx + 1);
            pc[p] = (uint8_t)(((vi - vj) % 3 + 3) % 3);
          }
          for (int cc = 0; cc < 3; ++cc) {
            SweepLists &S = L.col[cc];
            plan_sweep_ctas(P, pp, cp, ct, ex, &pc, cc);
            S.pp = pp;
            S.ncta = (int)ct.size();
            if (S.ncta) {
              S.cta_patch = dupload(cp, s);
              S.cta_type = dupload(ct, s);
            }
            plan_sweep_ctas(P, 8, cp, ct, ex, &pc, cc);
            S.ngrp8 = (int)ct.size();
            if (S.ngrp8) {
              S.grp_patch8 = dupload(cp, s);
              S.grp_type8 = dupload(ct, s);
            }
            if (L.sym_ok) {
              std::vector<int32_t> sl;
              int32_t qi = 0;
              for (int64_t p = 0; p < P.npatch; ++p)
                if (P.ptype[p] == L.sym_cls) {
                  if (pc[p] == cc) sl.push_back(qi);
                  ++qi;
                }
              S.nsym = (int64_t)sl.size();
              if (S.nsym) S.sym_list = dupload(sl, s);
            }
          }
          L.coloured = true;
        }
      }
      {
        // algorithmic flops of one sweep, per (patch, slab), of the solve the path runs:
        //   LU mode: 2 m^2 + 2 m_p^2 (LU solve + jump);
        //   Kronecker: 2 (2 (q+1) m_p^2 + m_p (q+1)^2) (two transforms + per-mode DG(q) solves);
        //   symmetric class: 2 (2 (q+1) sum_chi d_chi^2 + m_p (q+1)^2) (host_sym.cu blocks)
        const double nq = c->nq, s2 = degree == 3 ? 99.0 : 15.0;
        double fl = 0.0;
        for (int64_t p = 0; p < P.npatch; ++p) {
          const double ps = P.psize[p];
          if (!c->use_kron)
            fl += 2.0 * (nq * ps) * (nq * ps) + 2.0 * ps * ps;
          else if (L.sym_ok && P.ptype[p] == L.sym_cls)
            fl += 2.0 * (2.0 * nq * s2 + ps * nq * nq);
          else
            fl += 2.0 * (2.0 * nq * ps * ps + ps * nq * nq);
        }
        c->sweep_flops.push_back(fl * c->N);
      }
      if (l < nl - 1) {
        L.vr = dzalloc<double>(L.nnode * c->nt);
        L.vz = dzalloc<double>(L.nnode * c->nt);
        L.vt = dzalloc<double>(L.nnode * c->nt);
      }
      if (c->strip)
        for (int b = 0; b < 4; ++b) L.hx[b] = dalloc<double>((size_t)L.Ly * degree * c->nt);
      CK(cudaStreamSynchronize(s));  // host plan vectors die at scope end
    }
    for (int l = 1; l < nl; ++l) {
      std::vector<int32_t> rp, ci, trp, tci;
      std::vector<double> v, tv;
      if (c->strip)
        plan_strip_interpolation(plans[l - 1], c->lv[l - 1].st, plans[l], c->lv[l].st, degree, nys[l], rp, ci, v,
                                 neumann);
      else
        plan_interpolation(plans[l - 1], plans[l], degree, rp, ci, v);
      transpose_csr(plans[l].nnode, plans[l - 1].nnode, rp, ci, v, trp, tci, tv);
      Level &C = c->lv[l - 1];
      C.P.nrow = plans[l].nnode;
      C.P.nnz = (int64_t)ci.size();
      C.P.rowptr = dupload(rp, s);
      C.P.col = dupload(ci, s);
      C.P.val = dupload(v, s);
      C.R.nrow = plans[l - 1].nnode;
      C.R.nnz = (int64_t)tci.size();
      C.R.rowptr = dupload(trp, s);
      C.R.col = dupload(tci, s);
      C.R.val = dupload(tv, s);
      CK(cudaStreamSynchronize(s));
    }
    if (c->sub) {  // hand-over between the coarsest partitioned level and the replicated hierarchy
      const Level &T = c->sub->lv.back();
      PlanLevel gc;
      plan_level(T.nx, T.ny, T.h, degree, &gc, neumann);
      StripInfo whole{};
      whole.gnx = T.nx;
      whole.nx = T.nx;
      whole.nxl = T.nx;
      std::vector<int32_t> rp, ci, trp, tci;
      std::vector<double> v, tv;
      plan_strip_interpolation(gc, whole, plans[0], c->lv[0].st, degree, nys[0], rp, ci, v, neumann);
      transpose_csr(plans[0].nnode, gc.nnode, rp, ci, v, trp, tci, tv);
      Level &X = c->xfer;
      X.P.nrow = plans[0].nnode;
      X.P.nnz = (int64_t)ci.size();
      X.P.rowptr = dupload(rp, s);
      X.P.col = dupload(ci, s);
      X.P.val = dupload(v, s);
      X.R.nrow = gc.nnode;
      X.R.nnz = (int64_t)tci.size();
      X.R.rowptr = dupload(trp, s);
      X.R.col = dupload(tci, s);
      X.R.val = dupload(tv, s);
      const int64_t ng = gc.nnode * c->nt;
      c->sub_r = dzalloc<double>(ng);
      c->sub_z = dzalloc<double>(ng);
      c->sub_part = dzalloc<double>(ng);
      c->sub_all = dzalloc<double>(ng * coeffs->nranks);
      CK(cudaStreamSynchronize(s));
    }
    PlanLevel gplan;  // strips: the global coarsest level, replicated on every rank
    if (c->strip && !c->sub) {
      const double h0 = mesh->h * (double)(mesh->gnx / nxs[0]);
      plan_level(nxs[0], nys[0], h0, degree, &gplan, neumann);
      Level &G = c->gco;
      G.nx = gplan.nx;
      G.ny = gplan.ny;
      G.h = h0;
      G.Lx = gplan.Lx;
      G.Ly = gplan.Ly;
      G.nnode = gplan.nnode;
      G.nfree = gplan.nfree;
      G.A.nrow = gplan.nnode;
      G.A.nnz = (int64_t)gplan.col.size();
      G.A.rowptr = dupload(gplan.rowptr, s);
      G.A.col = dupload(gplan.col, s);
      G.A.val = dalloc<double>(gplan.col.size());
      G.A.val2 = dalloc<double>(gplan.col.size());
      G.h_con = gplan.con;
      G.con = dupload(gplan.con, s);
      c->gr = dalloc<double>(G.nnode * c->nt);
      c->gz = dalloc<double>(G.nnode * c->nt);
      c->gchunk = (int64_t)G.Ly * (degree * c->lv[0].st.nx + 1) * c->nt;
      c->gsend = dalloc<double>(c->gchunk);
      c->grecv = dalloc<double>(c->gchunk * coeffs->nranks);
      CK(cudaMemsetAsync(c->gr, 0, G.nnode * c->nt * sizeof(double), s));
      CK(cudaStreamSynchronize(s));
    }
    if (!c->sub) {
      const PlanLevel &CP = c->strip ? gplan : plans[0];
      Coarse &C = c->coarse;
      std::vector<int32_t> nodes;
      for (int64_t i = 0; i < CP.nnode; ++i)
        if (!CP.con[i]) nodes.push_back((int32_t)i);
      if (nodes.empty()) throw Err{WRMG_E_INVALID, "coarse level has no free node"};
      C.nfree = (int64_t)nodes.size();
      C.mp = (int)nodes.size();
      C.m = c->nq * C.mp;
      C.nodes = dupload(nodes, s);
      C.Dblk = dalloc<double>((size_t)C.m * C.m);
      C.DinvT = dalloc<double>((size_t)C.m * C.m);
      C.GT = dalloc<double>((size_t)C.m * C.mp);
      C.Gq = dalloc<double>((size_t)C.mp * C.mp);
      C.Z = dalloc<double>((size_t)c->N * C.m);
      C.Y = dalloc<double>((size_t)(c->N + 1) * C.mp);
      C.piv = dalloc<int32_t>(C.m);
      C.info = dalloc<int32_t>(1);
      // coarsest levels with more than kCoarseKronMax free nodes: the slab march with the
      // stored block inverse (the single-CTA Jacobi eigen-setup of the Kronecker form costs
      // O(mp^3) sweeps serially: minutes at mp = 841, the paper protocol's P3 10 x 10 level)
      c->coarse_kron = c->use_kron && C.mp <= kCoarseKronMax;
      if (c->coarse_kron) {
        C.kV = dalloc<double>((size_t)C.mp * C.mp);
        C.kVT = dalloc<double>((size_t)C.mp * C.mp);
        C.kS = dalloc<double>((size_t)C.mp * c->nq * c->nq);
        C.ksig = dalloc<double>((size_t)C.mp);
      }
    }
    c->tmp = dzalloc<double>(c->lv.back().nnode * c->nt);
    c->red = dalloc<double>(64 + 64 * kDotBlocksMax);
    CK(cudaStreamSynchronize(s));
    factor_all(c);
    c->cheb = coeffs->smoother == WRMG_SMOOTH_CHEBYSHEV;
    if (c->cheb) {
      if (c->co.cheb_steps == 0) c->co.cheb_steps = 50;
      c->lam.assign(nl, 0.0);
      c->cd.assign(nl, nullptr);
      c->cbr.assign(nl, nullptr);
      for (int l = c->sub ? 0 : 1; l < nl; ++l) {  // strips over a replicated sub-hierarchy: level 0 is smoothed
        c->cd[l] = dzalloc<double>(c->lv[l].nnode * c->nt);
        c->cbr[l] = dzalloc<double>(c->lv[l].nnode * c->nt);
        c->lam[l] = estimate_lambda(c, l);
      }
    }
    *out = c;
    return WRMG_OK;
  } catch (const Err &e) {
    wrmg_status st = fail(c, e);
    if (c) wrmg_destroy(c);
    return st;
  } catch (const std::bad_alloc &) {
    if (c) wrmg_destroy(c);
    g_err = "host allocation failed";
    return WRMG_E_OOM;
  }
}

wrmg_status wrmg_layout(const wrmg_ctx *c, wrmg_layout_t *out) {
  if (!c || !out) return WRMG_E_INVALID;
  const Level &L = c->lv.back();
  std::memset(out, 0, sizeof(*out));
  out->nnode = L.nnode;
  out->nt = c->nt;
  out->ndof = L.nnode * c->nt;
  out->nfree_st = L.nfree * c->nt;
  out->lx = L.Lx;
  out->ly = L.Ly;
  out->nlevels = (int)c->lv.size();
  out->degree = c->k;
  out->q = c->q;
  out->nslabs = c->N;
  out->npatch = L.npatch;
  out->mp_max = L.mp;
  out->npatch_types = L.ntypes;
  int64_t upd = 0;
  for (size_t l = 1; l < c->lv.size(); ++l) upd += c->lv[l].nfree * c->nt * (c->co.nu_pre + c->co.nu_post);
  out->smooth_dof_updates_per_vcycle = upd;
  out->own0 = L.st.own0;
  out->own1 = L.st.own1;
  out->g0 = L.st.G0;
  out->nfree_owned_st = L.nfree_owned * c->nt;
  if (c->ns) {
    out->lu = L.Lu;
    out->lpx = L.Lpx;
    out->lpy = (int32_t)(L.Lp / L.Lpx);
    out->own0p = L.stp.own0;
    out->own1p = L.stp.own1;
    out->g0p = L.stp.G0;
  }
  if (c->strip) {  // owned rows; the replicated levels (c->sub) are counted once, on rank 0
    upd = 0;
    for (size_t l = c->sub ? 0 : 1; l < c->lv.size(); ++l)
      upd += c->lv[l].nfree_owned * c->nt * (c->co.nu_pre + c->co.nu_post);
    if (c->sub) {
      out->nlevels += (int)c->sub->lv.size();
      if (c->co.rank == 0) {
        wrmg_layout_t sl;
        wrmg_layout(c->sub, &sl);
        upd += sl.smooth_dof_updates_per_vcycle;
      }
    }
    out->smooth_dof_updates_per_vcycle = upd;
  }
  return WRMG_OK;
}

wrmg_status wrmg_linearize(wrmg_ctx *c, const double *state) {
  if (!c || (state && !al16(state))) return WRMG_E_INVALID;
  DevGuard dg_(c, __func__);
  try {
    if (c->ns) {
      factor_all_ns(c, state);
      return WRMG_OK;
    }
    if (state) throw Err{WRMG_E_UNSUPPORTED, "heat operator is linear: state must be NULL"};
    factor_all(c);
    return WRMG_OK;
  } catch (const Err &e) {
    return fail(c, e);
  }
}

wrmg_status wrmg_rhs(wrmg_ctx *c, const double *fhat, double *b) {
  if (!c || !fhat || !b || !al16(fhat, b)) return WRMG_E_INVALID;
  DevGuard dg_(c, __func__);
  try {
    if (c->ns) {  // R6 (C3): b = drawn values on free rows, 0 on constrained rows, pressure mean-projected
      const Level &L = c->lv.back();
      launch_ns_mask(L.nnode, c->nt, L.con, nullptr, fhat, b, c->stream);
      ns_project(c, L, b);
      check_launch();
      return WRMG_OK;
    }
    launch_rhs(c->lv.back(), c->q, c->N, c->tm, fhat, b, c->stream);
    check_launch();
    return WRMG_OK;
  } catch (const Err &e) {
    return fail(c, e);
  }
}

wrmg_status wrmg_rhs_initial(wrmg_ctx *c, const double *u0, double *b) {
  if (!c || !u0 || !b || !al16(u0, b)) return WRMG_E_INVALID;
  DevGuard dg_(c, __func__);
  try {
    launch_rhs_initial(c->lv.back(), c->nq, c->nt, c->tm.phi0, u0, b, c->stream);
    check_launch();
    return WRMG_OK;
  } catch (const Err &e) {
    return fail(c, e);
  }
}

wrmg_status wrmg_set_boundary_values(wrmg_ctx *c, const double *g) {
  if (!c || (g && !al16(g))) return WRMG_E_INVALID;
  if (!c->ns) {
    c->err = "wrmg_set_boundary_values: Navier-Stokes contexts only";
    return WRMG_E_UNSUPPORTED;
  }
  DevGuard dg_(c, __func__);
  try {
    const int64_t n = c->lv.back().nnode * c->nt;
    if (!g) {
      if (c->bcg_st) CK(cudaFree(c->bcg_st));
      c->bcg_st = nullptr;
      return WRMG_OK;
    }
    if (!c->bcg_st) c->bcg_st = dalloc<double>(n);
    CK(cudaMemcpyAsync(c->bcg_st, g, n * sizeof(double), cudaMemcpyDefault, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    return WRMG_OK;
  } catch (const Err &e) {
    return fail(c, e);
  }
}

wrmg_status wrmg_cheb_lambda(const wrmg_ctx *c, int32_t level, double *lam) {
  if (!c || !lam || level < 0 || level >= (int)c->lv.size()) return WRMG_E_INVALID;
  *lam = c->cheb ? c->lam[level] : 0.0;
  return WRMG_OK;
}

wrmg_status wrmg_residual(wrmg_ctx *c, const double *u, const double *b, double *r, int32_t nonlinear) {
  if (!c || !u || !b || !r || !al16(u, b, r)) return WRMG_E_INVALID;
  if (nonlinear && !c->ns) return WRMG_E_UNSUPPORTED;
  DevGuard dg_(c, __func__);
  try {
    if (nonlinear) {
      if (c->strip) halo_forward(c, c->lv.back(), const_cast<double *>(u));
      ns_nonlinear_residual(c, u, b, r);
      check_launch();
      return WRMG_OK;
    }
    if (c->strip) halo_forward(c, c->lv.back(), const_cast<double *>(u));
    prof_residual(c, (int)c->lv.size() - 1, u, b, r, false);
    check_launch();
    return WRMG_OK;
  } catch (const Err &e) {
    return fail(c, e);
  }
}

wrmg_status wrmg_apply(wrmg_ctx *c, const double *x, double *y) {
  if (!c || !x || !y || !al16(x, y)) return WRMG_E_INVALID;
  DevGuard dg_(c, __func__);
  try {
    if (c->strip) halo_forward(c, c->lv.back(), const_cast<double *>(x));
    prof_residual(c, (int)c->lv.size() - 1, x, nullptr, y, false);  // b = NULL: y = A x
    check_launch();
    return WRMG_OK;
  } catch (const Err &e) {
    return fail(c, e);
  }
}

wrmg_status wrmg_smooth(wrmg_ctx *c, double *u, const double *b, int32_t nsweeps, double omega) {
  if (!c || !u || !b || nsweeps < 0 || !al16(u, b)) return WRMG_E_INVALID;
  DevGuard dg_(c, __func__);
  try {
    const int l = (int)c->lv.size() - 1;
    for (int s = 0; s < nsweeps; ++s) {
      if (c->strip) {
        halo_forward(c, c->lv[l], u);
        prof_residual(c, l, u, b, c->tmp, false);
        halo_forward(c, c->lv[l], c->tmp);
        sweep_strip(c, l, c->tmp, u, omega);
        continue;
      }
      prof_residual(c, l, u, b, c->tmp, false);
      prof_sweep(c, l, c->tmp, u, omega);
    }
    check_launch();
    return WRMG_OK;
  } catch (const Err &e) {
    return fail(c, e);
  }
}

wrmg_status wrmg_vcycle(wrmg_ctx *c, const double *r, double *z) {
  if (!c || !r || !z || !al16(r, z)) return WRMG_E_INVALID;
  DevGuard dg_(c, __func__);
  try {
    vcycle_level(c, (int)c->lv.size() - 1, r, z);
    check_launch();
    return WRMG_OK;
  } catch (const Err &e) {
    return fail(c, e);
  }
}

wrmg_status wrmg_level_size(const wrmg_ctx *c, int32_t level, int64_t *nnode) {
  if (!c || !nnode || level < 0 || level >= (int)c->lv.size()) return WRMG_E_INVALID;
  *nnode = c->lv[level].nnode;
  return WRMG_OK;
}

wrmg_status wrmg_restrict(wrmg_ctx *c, int32_t level, const double *rf, double *rc) {
  if (!c || !rf || !rc || level < 1 || level >= (int)c->lv.size() || !al16(rf, rc)) return WRMG_E_INVALID;
  DevGuard dg_(c, __func__);
  try {
    launch_restrict(c->lv[level - 1], c->nt, rf, rc, c->stream);
    check_launch();
    return WRMG_OK;
  } catch (const Err &e) {
    return fail(c, e);
  }
}

wrmg_status wrmg_prolong_add(wrmg_ctx *c, int32_t level, const double *ec, double *uf) {
  if (!c || !ec || !uf || level < 1 || level >= (int)c->lv.size() || !al16(ec, uf)) return WRMG_E_INVALID;
  DevGuard dg_(c, __func__);
  try {
    launch_prolong_add(c->lv[level - 1], c->nt, ec, uf, c->stream);
    check_launch();
    return WRMG_OK;
  } catch (const Err &e) {
    return fail(c, e);
  }
}

wrmg_status wrmg_fgmres(wrmg_ctx *c, const double *b, double *x, int32_t restart, int32_t maxit, double rtol,
                        double atol, int32_t *iters, double *relres) {
  if (!c || !b || !x || restart < 1 || restart > 31 || maxit < 1 || !al16(b, x)) return WRMG_E_INVALID;
  DevGuard dg_(c, __func__);
  try {
    cudaStream_t s = c->stream;
    Level &L = c->lv.back();
    const bool strip = c->strip;
    const bool cgs2 = c->co.orth == WRMG_ORTH_CGS2;
    const int64_t n = L.nnode * c->nt;
    if (c->restart_alloc < restart) {
      for (double *p : c->V) dfree(p);
      for (double *p : c->Z) dfree(p);
      c->V.clear();
      c->Z.clear();
      dfree(c->w);
      for (int i = 0; i <= restart; ++i) c->V.push_back(dzalloc<double>(n));
      for (int i = 0; i < restart; ++i) c->Z.push_back(dzalloc<double>(n));
      c->w = dzalloc<double>(n);
      c->restart_alloc = restart;
    }
    double *red = c->red;            // [0, 64): results / coefficients
    double *part = c->red + 64;      // partial sums
    auto norm = [&](const double *v) { return std::sqrt(dot_host(c, v, v, n)); };
    auto multidot = [&](int nv, const double *w, std::vector<double> &h) {
      int nb = multidot_blocks(n);
      std::vector<const double *> Vp(c->V.begin(), c->V.begin() + nv);
      {
        PScope ps(c, WRMG_K_KRYLOV, (int)c->lv.size() - 1, 8.0 * (nv + 1) * n, 2.0 * nv * n);
        launch_multidot(Vp.data(), nv, w, n, part, nb, s);
        launch_reduce_partials(part, nb, nv, red, s);
      }
      h.resize(nv);
      reduce_to_host(c, red, nv, h.data());
    };
    CK(cudaMemsetAsync(x, 0, n * sizeof(double), s));
    // strips: norms and dots over owned rows (ghost columns of the Krylov vectors are zero)
    const double bnorm = strip ? 0.0 : norm(b);
    double bnorm_g = bnorm;
    if (strip) {
      CK(cudaMemcpyAsync(c->tmp, b, n * sizeof(double), cudaMemcpyDeviceToDevice, s));
      zero_ghosts(c, L, c->tmp);
      bnorm_g = norm(c->tmp);
    }
    const double target = std::max(rtol * bnorm_g, atol);
    int its = 0;
    wrmg_status status = WRMG_E_NOT_CONVERGED;
    CK(cudaMemcpyAsync(c->tmp, b, n * sizeof(double), cudaMemcpyDeviceToDevice, s));  // r = b (x0 = 0)
    if (strip) zero_ghosts(c, L, c->tmp);
    double beta = strip ? norm(c->tmp) : bnorm;
    bool done = beta <= target;
    if (done) status = WRMG_OK;
    std::vector<double> H((size_t)(restart + 1) * restart), cs(restart), sn(restart), g(restart + 1), h, h2, y;
    // Lazily scaled basis: the stored V_i' and Z_i' = B V_i' carry a host scale sc_i
    // (V_i = sc_i V_i', sc_i = 1 / |V_i'|), so no pass over the vectors normalises
    // them: the new basis vector is the orthogonalised w itself (buffer swap) and
    // the scales enter the CGS coefficients, the Hessenberg entries and y.
    std::vector<double> sc(restart + 1, 0.0), coef(32);
    if (!strip && !c->kry) c->kry = dalloc<double>(256);
    while (!done && its < maxit) {
      std::swap(c->V[0], c->tmp);  // V_0' = r, sc_0 = 1 / beta
      sc[0] = 1.0 / beta;
      if (!strip) small_h2d(c, &sc[0], c->kry, 1);
      std::fill(H.begin(), H.end(), 0.0);
      std::fill(g.begin(), g.end(), 0.0);
      g[0] = beta;
      int jend = 0;
      for (int j = 0; j < restart; ++j) {
        vcycle_level(c, (int)c->lv.size() - 1, c->V[j], c->Z[j]);  // strips: z valid on owned + ghost columns
        if (strip) zero_ghosts(c, L, c->V[j]);  // the cycle refreshed V_j's ghosts; dots count owned rows only
        // w = A Z_j (residual kernel in apply mode)
        prof_residual(c, (int)c->lv.size() - 1, c->Z[j], nullptr, c->w, false);
        if (strip) zero_ghosts(c, L, c->w);
        // CGS (R16), fused: h = V^T w;  w -= V h & |w|^2.
        // CGS2, fused: h = V^T w;  w -= V h & h2 = V^T w;  w -= V h2 & |w|^2
        // (w' = A Z_j', the true w = sc_j w': h_i = sc_i sc_j <V_i', w'>, and
        // w -= sum h_i V_i  <=>  w' -= sum sc_i^2 <V_i', w'> V_i')
        double wn2 = 0.0;
        if (!strip) {  // coefficients on the device: one host read per Arnoldi step
          const int nb = multidot_blocks(n);
          std::vector<const double *> Vp(c->V.begin(), c->V.begin() + j + 1);
          {
            PScope ps(c, WRMG_K_KRYLOV, (int)c->lv.size() - 1, 8.0 * (j + 2) * n, 2.0 * (j + 1) * n);
            launch_multidot(Vp.data(), j + 1, c->w, n, part, nb, s);
            launch_reduce_partials(part, nb, j + 1, c->kry + 32, s);
          }
          launch_cgs_step(c->kry, j, 0, s);
          if (cgs2) {
            {
              PScope ps(c, WRMG_K_KRYLOV, (int)c->lv.size() - 1, 8.0 * (j + 3) * n, 4.0 * (j + 1) * n);
              launch_cgs_update_dot(c->V.data(), j + 1, c->w, c->kry + 64, n, part, nb, s);
              launch_reduce_partials(part, nb, j + 1, c->kry + 96, s);
            }
            launch_cgs_step(c->kry, j, 1, s);
          }
          {  // CGS: w -= V coef_A and |w|^2 in one pass (CGS2: coef_B)
            PScope ps(c, WRMG_K_KRYLOV, (int)c->lv.size() - 1, 8.0 * (j + 3) * n, 2.0 * (j + 2) * n);
            launch_cgs_update_norm(c->V.data(), j + 1, c->w, c->kry + (cgs2 ? 128 : 64), n, part, nb, s);
            launch_reduce_partials(part, nb, 1, c->kry + 192, s);
          }
          launch_cgs_step(c->kry, j, 2, s);
          std::vector<double> out(j + 2);
          small_d2h(c, c->kry + 200, out.data(), j + 2);
          h.assign(out.begin(), out.begin() + j + 1);
          wn2 = out[j + 1];
        } else {
        multidot(j + 1, c->w, h);
        for (int i = 0; i <= j; ++i) {
          coef[i] = sc[i] * sc[i] * h[i];
          h[i] *= sc[i] * sc[j];
        }
        if (!cgs2) {  // CGS: w -= V coef and |w|^2 in one pass
          small_h2d(c, coef.data(), red + 32, j + 1);
        } else {
        small_h2d(c, coef.data(), red, j + 1);
        {
          PScope ps(c, WRMG_K_KRYLOV, (int)c->lv.size() - 1, 8.0 * (j + 3) * n, 4.0 * (j + 1) * n);
          const int nb = multidot_blocks(n);
          launch_cgs_update_dot(c->V.data(), j + 1, c->w, red, n, part, nb, s);
          launch_reduce_partials(part, nb, j + 1, red + 32, s);
        }
        h2.resize(j + 1);
        reduce_to_host(c, red + 32, j + 1, h2.data());
        for (int i = 0; i <= j; ++i) {
          coef[i] = sc[i] * sc[i] * h2[i];
          h[i] += sc[i] * sc[j] * h2[i];
        }
        small_h2d(c, coef.data(), red + 32, j + 1);
        }
        {
          PScope ps(c, WRMG_K_KRYLOV, (int)c->lv.size() - 1, 8.0 * (j + 3) * n, 2.0 * (j + 2) * n);
          const int nb = multidot_blocks(n);
          launch_cgs_update_norm(c->V.data(), j + 1, c->w, red + 32, n, part, nb, s);
          launch_reduce_partials(part, nb, 1, red + 63, s);
        }
        reduce_to_host(c, red + 63, 1, &wn2);
        }
        const double hn = sc[j] * std::sqrt(wn2);
        std::vector<double> col(restart + 1, 0.0);
        for (int i = 0; i <= j; ++i) col[i] = h[i];
        col[j + 1] = hn;
        for (int i = 0; i < j; ++i) {
          double t = cs[i] * col[i] + sn[i] * col[i + 1];
          col[i + 1] = -sn[i] * col[i] + cs[i] * col[i + 1];
          col[i] = t;
        }
        const double d = std::hypot(col[j], col[j + 1]);
        cs[j] = col[j] / d;
        sn[j] = col[j + 1] / d;
        col[j] = d;
        col[j + 1] = 0.0;
        g[j + 1] = -sn[j] * g[j];
        g[j] = cs[j] * g[j];
        for (int i = 0; i <= restart; ++i) H[(size_t)i * restart + j] = col[i];
        ++its;
        jend = j + 1;
        if (hn < 1e-30) {
          status = WRMG_E_BREAKDOWN;
          done = true;
          break;
        }
        std::swap(c->V[j + 1], c->w);  // V_{j+1}' = w', sc_{j+1} = 1 / |w'|
        sc[j + 1] = 1.0 / std::sqrt(wn2);
        if (std::fabs(g[j + 1]) <= target) {
          status = WRMG_OK;
          done = true;
          break;
        }
        if (its >= maxit) {
          done = true;
          break;
        }
      }
      y.assign(jend, 0.0);
      for (int i = jend - 1; i >= 0; --i) {
        double acc = g[i];
        for (int k2 = i + 1; k2 < jend; ++k2) acc -= H[(size_t)i * restart + k2] * y[k2];
        y[i] = acc / H[(size_t)i * restart + i];
      }
      for (int i = 0; i < jend; ++i) y[i] *= sc[i];  // x += sum y_i Z_i = sum (y_i sc_i) Z_i'
      small_h2d(c, y.data(), red, jend);
      {
        PScope ps(c, WRMG_K_KRYLOV, (int)c->lv.size() - 1, 8.0 * (jend + 2) * n, 2.0 * jend * n);
        launch_multiaxpy(x, c->Z.data(), red, jend, n, 1.0, s);
      }
      CK(cudaStreamSynchronize(s));
      if (done) break;
      if (strip) halo_forward(c, L, x);
      prof_residual(c, (int)c->lv.size() - 1, x, b, c->tmp, false);
      if (strip) zero_ghosts(c, L, c->tmp);
      beta = norm(c->tmp);
      if (beta <= target) {
        status = WRMG_OK;
        break;
      }
    }
    if (strip) halo_forward(c, L, x);
    prof_residual(c, (int)c->lv.size() - 1, x, b, c->tmp, false);
    if (strip) zero_ghosts(c, L, c->tmp);
    const double rn = norm(c->tmp);
    if (iters) *iters = its;
    if (relres) *relres = bnorm_g > 0 ? rn / bnorm_g : 0.0;
    check_launch();
    if (status != WRMG_OK) c->err = status == WRMG_E_BREAKDOWN ? "FGMRES breakdown" : "FGMRES: maxit reached";
    return status;
  } catch (const Err &e) {
    return fail(c, e);
  }
}

wrmg_status wrmg_stationary(wrmg_ctx *c, const double *b, double *u, int32_t ncycles) {
  if (!c || !b || !u || ncycles < 0 || !al16(b, u)) return WRMG_E_INVALID;
  DevGuard dg_(c, __func__);
  try {
    const int top = (int)c->lv.size() - 1;
    const int64_t n = c->lv.back().nnode * c->nt;
    if (!c->st_r) {
      c->st_r = dzalloc<double>(n);
      c->st_z = dzalloc<double>(n);
    }
    for (int it = 0; it < ncycles; ++it) {
      if (c->strip) halo_forward(c, c->lv.back(), u);
      prof_residual(c, top, u, b, c->st_r, false);
      if (c->ns) ns_project(c, c->lv.back(), c->st_r);
      vcycle_level(c, top, c->st_r, c->st_z);
      launch_axpy(n, 1.0, c->st_z, u, c->stream);  // strips: z valid on owned and ghost columns
    }
    check_launch();
    return WRMG_OK;
  } catch (const Err &e) {
    return fail(c, e);
  }
}

wrmg_status wrmg_fgmres_host(wrmg_ctx *c, int32_t nrhs, const double *const *b_host, double *const *x_host,
                             int32_t restart, int32_t maxit, double rtol, double atol, int32_t *iters,
                             double *relres) {
  if (!c || nrhs < 0 || (nrhs > 0 && (!b_host || !x_host))) return WRMG_E_INVALID;
  DevGuard dg_(c, __func__);
  try {
    const int64_t n = c->lv.back().nnode * c->nt;
    const size_t bytes = (size_t)n * sizeof(double);
    if (!c->copy) {
      CK(cudaStreamCreateWithFlags(&c->copy, cudaStreamNonBlocking));
      for (int j = 0; j < 2; ++j) {
        c->hb[j] = dalloc<double>(n);
        c->hx[j] = dalloc<double>(n);
        CK(cudaEventCreateWithFlags(&c->ev_in[j], cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&c->ev_solved[j], cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&c->ev_out[j], cudaEventDisableTiming));
      }
    }
    cudaStream_t s = c->stream, cs = c->copy;
    wrmg_status first = WRMG_OK;
    auto upload = [&](int i) {
      const int j = i & 1;
      if (i >= 2) CK(cudaStreamWaitEvent(cs, c->ev_solved[j], 0));  // solve i-2 no longer reads hb[j]
      CK(cudaMemcpyAsync(c->hb[j], b_host[i], bytes, cudaMemcpyHostToDevice, cs));
      CK(cudaEventRecord(c->ev_in[j], cs));
    };
    if (nrhs > 0) upload(0);
    for (int i = 0; i < nrhs; ++i) {
      const int j = i & 1;
      if (i + 1 < nrhs) upload(i + 1);  // on the copy engines while i is solved
      CK(cudaStreamWaitEvent(s, c->ev_in[j], 0));
      if (i >= 2) CK(cudaStreamWaitEvent(s, c->ev_out[j], 0));  // x_{i-2} downloaded from hx[j]
      int32_t it = 0;
      double rr = 0.0;
      const wrmg_status st = wrmg_fgmres(c, c->hb[j], c->hx[j], restart, maxit, rtol, atol, &it, &rr);
      if (st != WRMG_OK && st != WRMG_E_NOT_CONVERGED && st != WRMG_E_BREAKDOWN) return st;
      if (st != WRMG_OK && first == WRMG_OK) first = st;
      if (iters) iters[i] = it;
      if (relres) relres[i] = rr;
      CK(cudaEventRecord(c->ev_solved[j], s));
      CK(cudaStreamWaitEvent(cs, c->ev_solved[j], 0));
      CK(cudaMemcpyAsync(x_host[i], c->hx[j], bytes, cudaMemcpyDeviceToHost, cs));
      CK(cudaEventRecord(c->ev_out[j], cs));
    }
    CK(cudaStreamSynchronize(cs));
    CK(cudaStreamSynchronize(s));
    return first;
  } catch (const Err &e) {
    return fail(c, e);
  }
}

wrmg_status wrmg_profile(wrmg_ctx *c, int32_t enable) {
  if (!c) return WRMG_E_INVALID;
  DevGuard dg_(c, __func__);
  try {
    CK(cudaStreamSynchronize(c->stream));
    for (auto &r : c->prof_recs) {
      c->prof_pool.push_back(r.a);
      c->prof_pool.push_back(r.b);
    }
    c->prof_recs.clear();
    std::memset(c->stats, 0, sizeof(c->stats));
    c->prof_on = enable != 0;
    return WRMG_OK;
  } catch (const Err &e) {
    return fail(c, e);
  }
}

wrmg_status wrmg_kernel_stats(wrmg_ctx *c, wrmg_kernel_stat *out) {
  if (!c || !out) return WRMG_E_INVALID;
  DevGuard dg_(c, __func__);
  try {
    CK(cudaStreamSynchronize(c->stream));
    for (auto &r : c->prof_recs) {
      float ms = 0.f;
      CK(cudaEventElapsedTime(&ms, r.a, r.b));
      wrmg_kernel_stat &st = c->stats[r.cls][r.lvl];
      st.launches += 1;
      st.ms += ms;
      st.bytes += r.bytes;
      st.flops += r.flops;
      c->prof_pool.push_back(r.a);
      c->prof_pool.push_back(r.b);
    }
    c->prof_recs.clear();
    for (size_t l = 0; l < c->lv.size(); ++l)
      for (int k2 = 0; k2 < WRMG_K_COUNT; ++k2) out[l * WRMG_K_COUNT + k2] = c->stats[k2][l];
    return WRMG_OK;
  } catch (const Err &e) {
    return fail(c, e);
  }
}

int64_t wrmg_launch_count(void) { return g_launches.load(); }
int64_t wrmg_guard_violations(void) { return g_guard_violations.load(); }

wrmg_status wrmg_hessenberg_eig(const double *H, int32_t n, double *wr, double *wi) {
  if (!H || !wr || !wi || n < 1) return WRMG_E_INVALID;
  std::vector<double> a(H, H + (size_t)n * n), r, i;
  if (!hessenberg_eigenvalues(a, n, r, i)) return WRMG_E_NOT_CONVERGED;
  for (int k = 0; k < n; ++k) {
    wr[k] = r[k];
    wi[k] = i[k];
  }
  return WRMG_OK;
}

wrmg_status wrmg_nccl_unique_id(void *out128) {
  if (!out128) return WRMG_E_INVALID;
  std::string e;
  if (!nccl_get_unique_id(out128, e)) {
    g_err = e;
    return WRMG_E_NCCL;
  }
  return WRMG_OK;
}

wrmg_status wrmg_loopback_create(int32_t nranks, void **hub) {
  if (!hub || nranks < 1) return WRMG_E_INVALID;
  *hub = loop_hub_create(nranks);
  return WRMG_OK;
}

void wrmg_loopback_destroy(void *hub) { loop_hub_destroy(hub); }

wrmg_status wrmg_debug_fetch(wrmg_ctx *c, int32_t level, int32_t which, void *host_dst, int64_t count) {
  if (!c || !host_dst || count < 0 || level < 0 || level >= (int)c->lv.size()) return WRMG_E_INVALID;
  DevGuard dg_(c, __func__);
  try {
    const Level &L = c->lv[level];
    const void *src = nullptr;
    int64_t avail = 0, esz = 8;
    switch (which) {
      case 0: src = L.A.val; avail = L.A.nnz; break;
      case 1: src = L.A.val2; avail = L.A.nnz; break;
      case 2: src = L.conv; avail = L.nvv * c->nt; break;
      case 3: src = L.state; avail = L.state ? L.nnode * c->nt : 0; break;
      case 4: src = c->coarse.nsD; avail = c->coarse.nsD ? (int64_t)c->N * c->coarse.m * c->coarse.m : 0; break;
      case 5: src = L.A.rowptr; avail = L.A.nrow + 1; esz = 4; break;
      case 6: src = L.A.col; avail = L.A.nnz; esz = 4; break;
      case 7: src = c->coarse.nodes; avail = c->coarse.nfree; esz = 4; break;
      case 8: src = c->coarse.nsinfo; avail = c->coarse.nsinfo ? c->N : 0; esz = 4; break;
      case 9: src = c->coarse.nspiv; avail = c->coarse.nspiv ? (int64_t)c->N * c->coarse.m : 0; esz = 4; break;
      default: return WRMG_E_INVALID;
    }
    if (!src || count > avail) return WRMG_E_INVALID;
    CK(cudaStreamSynchronize(c->stream));
    CK(cudaMemcpy(host_dst, src, count * esz, cudaMemcpyDeviceToHost));
    return WRMG_OK;
  } catch (const Err &e) {
    return fail(c, e);
  }
}

// Eisenstat-Walker choice 2 with safeguard (R22).
static double eisenstat_walker(double eta_prev, double fn, double fprev) {
  const double gamma = 1.0, alpha = 0.5 * (1.0 + std::sqrt(5.0)), eta_max = 0.9;
  double eta = gamma * std::pow(fn / fprev, alpha);
  const double sg = gamma * std::pow(eta_prev, alpha);
  if (sg > 0.1) eta = std::max(eta, sg);
  return std::min(eta, eta_max);
}

wrmg_status wrmg_newton(wrmg_ctx *c, double *U, double rtol, int32_t maxit, int32_t *newton_its, int32_t *lin_its) {
  return wrmg_newton_rhs(c, U, nullptr, rtol, maxit, newton_its, lin_its);
}

wrmg_status wrmg_newton_rhs(wrmg_ctx *c, double *U, const double *rhs, double rtol, int32_t maxit, int32_t *newton_its,
                            int32_t *lin_its) {
  if (!c || !U || maxit < 0) return WRMG_E_INVALID;
  if (!c->ns) {
    c->err = "wrmg_newton: the heat operator is linear";
    return WRMG_E_UNSUPPORTED;
  }
  if (!al16(U) || (rhs && !al16(rhs))) return WRMG_E_INVALID;
  DevGuard dg_(c, __func__);
  try {
    cudaStream_t s = c->stream;
    Level &L = c->lv.back();
    const int64_t n = L.nnode * c->nt;
    if (!c->nl_b) {
      c->nl_b = dalloc<double>(n);
      c->nl_r = dalloc<double>(n);
      c->nl_dx = dalloc<double>(n);
    }
    // Dirichlet / lid values on the constrained rows of U and of the residual's b (R5)
    launch_ns_mask(L.nnode, c->nt, L.con, c->bcg, U, U, s, c->bcg_st);
    launch_ns_mask(L.nnode, c->nt, L.con, c->bcg, rhs, c->nl_b, s, c->bcg_st);  // F(U) = rhs on free rows, U = g on constrained
    auto negF = [&]() {  // nl_r = -F(U)
      if (c->strip) halo_forward(c, L, U);
      ns_nonlinear_residual(c, U, c->nl_b, c->nl_r);
      if (c->strip) zero_ghosts(c, L, c->nl_r);  // norms over owned rows
      return std::sqrt(dot_host(c, c->nl_r, c->nl_r, n));
    };
    const double f0 = negF();
    double fn = f0, fprev = f0, eta = 0.3;
    int its = 0, lin = 0;
    for (int it = 0; it < maxit; ++it) {
      if (fn <= rtol * f0) break;
      factor_all_ns(c, U);
      ns_project(c, L, c->nl_r);
      int32_t li = 0;
      double rr = 0.0;
      wrmg_status st = wrmg_fgmres(c, c->nl_r, c->nl_dx, 30, 200, eta, 0.0, &li, &rr);
      if (st != WRMG_OK && st != WRMG_E_NOT_CONVERGED && st != WRMG_E_BREAKDOWN) return st;
      lin += li;
      ++its;
      launch_axpy(n, 1.0, c->nl_dx, U, s);
      ns_project(c, L, U);
      const double fnew = negF();
      eta = eisenstat_walker(eta, fnew, fprev);
      fprev = fnew;
      fn = fnew;
    }
    check_launch();
    CK(cudaStreamSynchronize(s));
    if (newton_its) *newton_its = its;
    if (lin_its) *lin_its = lin;
    if (!(fn <= rtol * f0)) {
      c->err = "Newton: maxit reached";
      return WRMG_E_NOT_CONVERGED;
    }
    return WRMG_OK;
  } catch (const Err &e) {
    return fail(c, e);
  }
}

wrmg_status wrmg_batched_lu(const wrmg_ctx *c, double *A, int32_t m, int32_t batch, int32_t *piv, int32_t *info) {
  if (!A || !piv || !info || m < 1 || batch < 0) return WRMG_E_INVALID;
  DevGuard dg_(c, __func__);
  try {
    cudaStream_t s = c ? c->stream : nullptr;
    launch_batched_lu(A, m, batch, piv, info, s);
    check_launch();
    CK(cudaStreamSynchronize(s));
    std::vector<int32_t> h(batch);
    if (batch) CK(cudaMemcpy(h.data(), info, batch * sizeof(int32_t), cudaMemcpyDeviceToHost));
    for (int32_t v : h)
      if (v) {
        g_err = "singular matrix in batched LU";
        return WRMG_E_SINGULAR;
      }
    return WRMG_OK;
  } catch (const Err &e) {
    return fail(nullptr, e);
  }
}

wrmg_status wrmg_fill_uniform(const wrmg_ctx *c, double *out, int64_t count, uint64_t first_id, uint64_t seed) {
  if (!out || count < 0) return WRMG_E_INVALID;
  DevGuard dg_(c, __func__);
  try {
    launch_fill_uniform(out, count, first_id, seed, c ? c->stream : nullptr);
    check_launch();
    return WRMG_OK;
  } catch (const Err &e) {
    return fail(nullptr, e);
  }
}

wrmg_status wrmg_sync(wrmg_ctx *c) {
  if (!c) return WRMG_E_INVALID;
  DevGuard dg_(c, __func__);
  try {
    CK(cudaStreamSynchronize(c->stream));
    check_launch();
    return WRMG_OK;
  } catch (const Err &e) {
    return fail(c, e);
  }
}

const char *wrmg_last_error(const wrmg_ctx *c, int32_t *level, int32_t *patch, int32_t *slab) {
  if (level) *level = c ? c->err_level : -1;
  if (patch) *patch = c ? c->err_patch : -1;
  if (slab) *slab = c ? c->err_slab : -1;
  if (c && !c->err.empty()) return c->err.c_str();
  return g_err.c_str();
}

void wrmg_destroy(wrmg_ctx *c) {
  if (!c) return;
  DevGuard dg_(c, __func__);
  if (c->stream) cudaStreamSynchronize(c->stream);
  dfree(c->st_r);
  dfree(c->st_z);
  if (c->copy) {
    cudaStreamSynchronize(c->copy);
    cudaStreamDestroy(c->copy);
    for (int j = 0; j < 2; ++j) {
      dfree(c->hb[j]);
      dfree(c->hx[j]);
      cudaEventDestroy(c->ev_in[j]);
      cudaEventDestroy(c->ev_solved[j]);
      cudaEventDestroy(c->ev_out[j]);
    }
  }
  if (c->side) {
    cudaStreamSynchronize(c->side);
    cudaStreamDestroy(c->side);
    cudaEventDestroy(c->ev_fork);
    cudaEventDestroy(c->ev_join);
  }
  if (c->hmap) cudaFreeHost(c->hmap);
  c->hmap = nullptr;
  for (auto &L : c->lv) free_level(L);
  free_level(c->gco);
  free_level(c->xfer);
  for (void *p : {(void *)c->sub_r, (void *)c->sub_z, (void *)c->sub_part, (void *)c->sub_all, (void *)c->sub_w,
                  (void *)c->rf_send, (void *)c->rf_recv, (void *)c->pj_sums, (void *)c->pj_all})
    dfree(p);
  if (c->sub) wrmg_destroy(c->sub);
  for (double *p : c->cd) dfree(p);
  for (double *p : c->cbr) dfree(p);
  for (void *p : {(void *)c->gr, (void *)c->gz, (void *)c->gsend, (void *)c->grecv}) dfree(p);
  delete c->comm;
  Coarse &C = c->coarse;
  for (void *p : {(void *)C.nodes, (void *)C.Dblk, (void *)C.DinvT, (void *)C.GT, (void *)C.Gq, (void *)C.Z,
                  (void *)C.Y, (void *)C.piv, (void *)C.info, (void *)C.kV, (void *)C.kVT, (void *)C.kS,
                  (void *)C.ksig, (void *)C.nsD, (void *)C.nsinvT, (void *)C.xq, (void *)C.nspiv, (void *)C.nsinfo,
                  (void *)C.nsH, (void *)C.nsG, (void *)C.nsZ, (void *)C.nsY, (void *)C.sid2c})
    dfree(p);
  for (void *p : {(void *)c->th_ref, (void *)c->th_T, (void *)c->bcg, (void *)c->bcg_st, (void *)c->gred, (void *)c->proj, (void *)c->conv_nl,
                  (void *)c->nl_b, (void *)c->nl_r, (void *)c->nl_dx})
    dfree(p);
  for (double *p : c->V) dfree(p);
  for (double *p : c->Z) dfree(p);
  dfree(c->w);
  dfree(c->red);
  dfree(c->kry);
  dfree(c->tmp);
  dfree(c->ref_dev);
  for (auto &r : c->prof_recs) {
    cudaEventDestroy(r.a);
    cudaEventDestroy(r.b);
  }
  for (cudaEvent_t e : c->prof_pool) cudaEventDestroy(e);
  delete c;
}

}  // extern "C"
