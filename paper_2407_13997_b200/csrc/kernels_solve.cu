// Hot-path kernels: space-time residual (H6), waveform-relaxation patch sweep
// with weighted additive scatter (H7 + H8), restriction / prolongation (H9,
// H10), coarse time-marching solve (H11), RHS assembly, RNG.
#include <algorithm>

#include <cstdlib>

#include "internal.h"

namespace wrmg {
namespace {

struct TMc {
  double CE[16], Mt[16];
};
TMc make_tmc(const Temporal &T) {
  TMc t{};
  for (int e = 0; e < T.nq * T.nq; ++e) {
    t.CE[e] = T.CE[e];
    t.Mt[e] = T.Mt[e];
  }
  return t;
}

// ------------------------------------------------------------------ residual
// r_n = b_n - [(C+E0) (x) M + Mt (x) kappa K] u_n + (E1 (x) M) u_{n-1}
// (eq. heatfem; R1, R3), constrained rows r = b - u (R5).
// A CTA owns an 8x8 tile of lattice rows and a chunk of 16 slabs; the u values of
// the tile plus a k-wide halo (every CSR neighbour of a tile row) are staged in
// shared memory once, so each u value is read from L2 once per tile instead of
// once per row that references it.  The slab chunk carries one extra value per
// node: u[node][n0-1][q], the upwind trace for the jump of the first slab.
constexpr int RT = 8;   // tile rows per direction
constexpr int RCS = 16; // slabs per chunk

template <int NQ>
__global__ void __launch_bounds__(256) k_residual(int k, int Lx, int Ly, int N, const int32_t *__restrict__ rowptr,
                                                  const int32_t *__restrict__ col, const double *__restrict__ Mv,
                                                  const double *__restrict__ Kv, const uint8_t *__restrict__ con,
                                                  const double *__restrict__ u, const double *__restrict__ b,
                                                  double *__restrict__ r, TMc tm) {
  extern __shared__ double su[];
  constexpr int W = RCS * NQ + 1;
  const int64_t NT = (int64_t)N * NQ;
  const int ntx = (Lx + RT - 1) / RT;
  const int tx0 = (blockIdx.x % ntx) * RT, ty0 = (blockIdx.x / ntx) * RT;
  const int n0 = blockIdx.y * RCS;
  const int nS = min(RCS, N - n0);
  const int RW = RT + 2 * k, RH = RT + 2 * k;
  const int tid = threadIdx.x;
  // stage u (region x chunk) in shared memory
  const int nreg = RW * RH;
  for (int e = tid; e < nreg * W; e += blockDim.x) {
    int node = e / W, off = e % W;
    int I = tx0 - k + node % RW, J = ty0 - k + node / RW;
    double v = 0.0;
    if (I >= 0 && I < Lx && J >= 0 && J < Ly) {
      const double *src = u + ((int64_t)J * Lx + I) * NT + (int64_t)n0 * NQ;
      if (off == 0) {
        if (n0 > 0) v = src[-1];
      } else if (off - 1 < nS * NQ) {
        v = src[off - 1];
      }
    }
    su[e] = v;
  }
  __syncthreads();
  const int s = tid & (RCS - 1), rg = tid >> 4;
  if (s >= nS) return;
  const int n = n0 + s;
  for (int rr = rg; rr < RT * RT; rr += 16) {
    const int I = tx0 + rr % RT, J = ty0 + rr / RT;
    if (I >= Lx || J >= Ly) continue;
    const int64_t i = (int64_t)J * Lx + I;
    const int64_t base = i * NT + (int64_t)n * NQ;
    if (con[i]) {
      const double *ul = su + ((J - ty0 + k) * RW + (I - tx0 + k)) * W + 1 + s * NQ;
#pragma unroll
      for (int a = 0; a < NQ; ++a) r[base + a] = b ? b[base + a] - ul[a] : ul[a];
      continue;
    }
    double am[NQ], ak[NQ], ap = 0.0;
#pragma unroll
    for (int a = 0; a < NQ; ++a) am[a] = ak[a] = 0.0;
    const int e1 = rowptr[i + 1];
    for (int e = rowptr[i]; e < e1; ++e) {
      const int j = __ldg(col + e);
      const double mv = __ldg(Mv + e), kv = __ldg(Kv + e);
      const int jI = j % Lx, jJ = j / Lx;
      const double *ul = su + ((jJ - ty0 + k) * RW + (jI - tx0 + k)) * W + s * NQ;
      ap = fma(mv, ul[0], ap);  // u[j][n-1][q] (slot 0 for s == 0)
#pragma unroll
      for (int a = 0; a < NQ; ++a) {
        am[a] = fma(mv, ul[1 + a], am[a]);
        ak[a] = fma(kv, ul[1 + a], ak[a]);
      }
    }
#pragma unroll
    for (int a = 0; a < NQ; ++a) {
      double acc = b ? b[base + a] : 0.0;
#pragma unroll
      for (int c = 0; c < NQ; ++c) acc -= tm.CE[a * NQ + c] * am[c] + tm.Mt[a * NQ + c] * ak[c];
      if (a == 0 && n > 0) acc += ap;  // (E1 (x) M) u_{n-1}: E1 = e_0 e_q^T (R2)
      r[base + a] = b ? acc : -acc;    // b == NULL: y = A u
    }
  }
}

// --------------------------------------------------------------------- sweep
// H7 + H8 for time-invariant patch blocks (heat).  One warp per patch, lanes =
// slabs of a 32-slab chunk (waveform-major gathers are 32 x (q+1) contiguous
// doubles per patch node).  With D the patch block, M_p its mass block and
// y_n = x_n[a = q] the end trace carried by the upwind jump (E1 = e_0 e_q^T):
//     x_n = D^{-1} (g_n + e_0 (x) M_p y_{n-1}) = z_n + G y_{n-1},
//     z_n = D^{-1} g_n,   G = D^{-1}[:, a=0] M_p          (forward sweep)
// z for the whole chunk is slab-parallel; only the m_p-long end trace recurs:
//     y_n = z_n[q] + G_q y_{n-1}    (sequential in n, lanes = patch rows).
// Scatter: u += omega / mu_i x (R11) with FP64 atomics (conflicts only between
// overlapping patches; the order of the <= 3 additions per value is the only
// nondeterminism).
constexpr int SW_WARPS = 4;

template <int NQ, int MP>
__global__ void __launch_bounds__(128) k_sweep(int64_t npatch, int N, const int32_t *__restrict__ pnodes,
                                               const int32_t *__restrict__ ptype, const double *__restrict__ Dinv,
                                               const double *__restrict__ Gm, const double *__restrict__ wnode,
                                               double omega, const double *__restrict__ r, double *__restrict__ u) {
  constexpr int M = NQ * MP;
  constexpr int ZS = 33;  // padded z row stride (bank spread for the lane = row reads)
  constexpr int SMW = M * ZS + 33 * MP + MP;
  extern __shared__ double sm[];
  __shared__ int s_nodes[SW_WARPS][MP];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t p = (int64_t)blockIdx.x * SW_WARPS + w;
  if (p >= npatch) return;
  double *zs = sm + w * SMW;
  double *ys = zs + M * ZS;
  double *ws = ys + 33 * MP;
  const int64_t NT = (int64_t)N * NQ;
  for (int j = lane; j < MP; j += 32) {
    int nd = pnodes[p * MP + j];
    s_nodes[w][j] = nd;
    ws[j] = nd >= 0 ? omega * wnode[nd] : 0.0;
    ys[j] = 0.0;
  }
  __syncwarp();
  const int ty = ptype[p];
  const double *Di = Dinv + (int64_t)ty * M * M;
  const double *Gt = Gm + (int64_t)ty * M * MP;
  for (int n0 = 0; n0 < N; n0 += 32) {
    const int S = min(32, N - n0);
    const int n = n0 + lane;
    const bool valid = lane < S;
    double g[M];
#pragma unroll
    for (int j = 0; j < MP; ++j) {
      const int nd = s_nodes[w][j];
      const double *src = r + (int64_t)nd * NT + (int64_t)n * NQ;
#pragma unroll
      for (int a = 0; a < NQ; ++a) g[a * MP + j] = (nd >= 0 && valid) ? __ldg(src + a) : 0.0;
    }
#pragma unroll
    for (int rho = 0; rho < M; ++rho) {
      double acc = 0.0;
      if constexpr (M % 2 == 0) {
        const double2 *drow = reinterpret_cast<const double2 *>(Di + rho * M);
#pragma unroll
        for (int s2 = 0; s2 < M / 2; ++s2) {
          const double2 d = __ldg(drow + s2);
          acc = fma(d.x, g[2 * s2], acc);
          acc = fma(d.y, g[2 * s2 + 1], acc);
        }
      } else {
#pragma unroll
        for (int sg = 0; sg < M; ++sg) acc = fma(__ldg(Di + rho * M + sg), g[sg], acc);
      }
      zs[rho * ZS + lane] = acc;
    }
    __syncwarp();
    {
      // all 32 lanes run the loop so every __syncwarp is full-mask
      const int row = lane < MP ? lane : 0;
      double gq[MP];
#pragma unroll
      for (int j = 0; j < MP; ++j) gq[j] = __ldg(Gt + ((NQ - 1) * MP + row) * MP + j);
      for (int st = 0; st < S; ++st) {
        double acc = zs[((NQ - 1) * MP + row) * ZS + st];
#pragma unroll
        for (int j = 0; j < MP; ++j) acc = fma(gq[j], ys[st * MP + j], acc);
        __syncwarp();
        if (lane < MP) ys[(st + 1) * MP + lane] = acc;
        __syncwarp();
      }
    }
    if (valid) {
      double yp[MP];
#pragma unroll
      for (int j = 0; j < MP; ++j) yp[j] = ys[lane * MP + j];
#pragma unroll
      for (int i = 0; i < MP; ++i) {
        const int nd = s_nodes[w][i];
        if (nd < 0) continue;
        double *dst = u + (int64_t)nd * NT + (int64_t)n * NQ;
        const double wi = ws[i];
#pragma unroll
        for (int a = 0; a < NQ - 1; ++a) {
          double x = zs[(a * MP + i) * ZS + lane];
#pragma unroll
          for (int j = 0; j < MP; ++j) x = fma(__ldg(Gt + (a * MP + i) * MP + j), yp[j], x);
          atomicAdd(dst + a, wi * x);
        }
        atomicAdd(dst + NQ - 1, wi * ys[(lane + 1) * MP + i]);
      }
    }
    __syncwarp();
    double c = 0.0;
    if (lane < MP) c = ys[S * MP + lane];
    __syncwarp();
    if (lane < MP) ys[lane] = c;
    __syncwarp();
  }
}

template <int NQ, int MP>
void sweep_launch(const Level &L, int N, const double *r, double *u, double omega, cudaStream_t s) {
  constexpr int M = NQ * MP;
  size_t smem = (size_t)SW_WARPS * (M * 33 + 33 * MP + MP) * sizeof(double);
  smem_optin((const void *)k_sweep<NQ, MP>, (int)smem);
  int blocks = (int)((L.npatch + SW_WARPS - 1) / SW_WARPS);
  k_sweep<NQ, MP><<<blocks, 32 * SW_WARPS, smem, s>>>(L.npatch, N, L.pnodes, L.ptype, L.Dinv, L.G, L.wnode, omega,
                                                      r, u); ++g_launches;
}

// ------------------------------------------------------------------ transfers
// H10: u_f += (P_h (x) I) e_c;  H9: r_c = (P_h^T (x) I) r_f.
template <bool ACC>
__global__ void __launch_bounds__(256) k_spmv_nt(int64_t nrow, int64_t NT2, const int32_t *__restrict__ rp,
                                                 const int32_t *__restrict__ ci, const double *__restrict__ v,
                                                 const double2 *__restrict__ x, double2 *__restrict__ y) {
  // thread = (row, pair of consecutive time values); NT even (checked by the launcher)
  const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (idx >= nrow * NT2) return;
  const int64_t i = idx / NT2, t = idx - i * NT2;
  const int e0 = rp[i], e1 = rp[i + 1];
  if (ACC && e0 == e1) return;
  double2 acc = make_double2(0.0, 0.0);
  double2 o = ACC ? y[idx] : make_double2(0.0, 0.0);  // loaded ahead of the gather loop
#pragma unroll 4
  for (int e = e0; e < e1; ++e) {
    const double a = __ldg(v + e);
    const double2 xv = __ldg(x + (int64_t)__ldg(ci + e) * NT2 + t);
    acc.x = fma(a, xv.x, acc.x);
    acc.y = fma(a, xv.y, acc.y);
  }
  if (ACC) {
    o.x += acc.x;
    o.y += acc.y;
    y[idx] = o;
  } else {
    y[idx] = acc;
  }
}

__global__ void k_spmv_nt1(int64_t nrow, int64_t NT, const int32_t *__restrict__ rp, const int32_t *__restrict__ ci,
                           const double *__restrict__ v, const double *__restrict__ x, double *__restrict__ y,
                           int accumulate) {
  int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (idx >= nrow * NT) return;
  int64_t i = idx / NT, t = idx - i * NT;
  double acc = 0.0;
  for (int e = rp[i]; e < rp[i + 1]; ++e) acc = fma(__ldg(v + e), __ldg(x + (int64_t)__ldg(ci + e) * NT + t), acc);
  if (accumulate) {
    if (rp[i + 1] > rp[i]) y[idx] += acc;
  } else {
    y[idx] = acc;
  }
}

// Same with each thread on TP pairs spaced NT2 / TP apart (NT2 % TP == 0): the row's
// index and value loads are shared by TP gathers, TP 16-byte loads in flight per entry.
// The kernel is latency-bound, so registers are capped for occupancy (measured on C2's finest
// level): prolongation (ACC) 4 CTAs/SM with the entry loop unrolled twice,
// restriction 5 CTAs/SM without unrolling.
template <bool ACC, int TP>
__global__ void __launch_bounds__(256, ACC ? 4 : 5) k_spmv_nt_tp(int64_t nrow, int64_t NT2, const int32_t *__restrict__ rp,
                                                    const int32_t *__restrict__ ci, const double *__restrict__ v,
                                                    const double2 *__restrict__ x, double2 *__restrict__ y) {
  const int64_t W = NT2 / TP;
  const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (idx >= nrow * W) return;
  const int64_t i = idx / W, t = idx - i * W;
  const int e0 = __ldg(rp + i), e1 = __ldg(rp + i + 1);
  if (ACC && e0 == e1) return;
  double2 acc[TP];
#pragma unroll
  for (int p = 0; p < TP; ++p) acc[p] = make_double2(0.0, 0.0);
  double2 *yr = y + i * NT2 + t;
  double2 yo[TP];  // ACC: the row's old values, loaded ahead of the gather loop
#pragma unroll
  for (int p = 0; p < TP; ++p) yo[p] = ACC ? yr[p * W] : make_double2(0.0, 0.0);
  constexpr int kTpUnroll = ACC ? 2 : 1;
#pragma unroll kTpUnroll
  for (int e = e0; e < e1; ++e) {
    const double a = __ldg(v + e);
    const double2 *xr = x + (int64_t)__ldg(ci + e) * NT2 + t;
#pragma unroll
    for (int p = 0; p < TP; ++p) {
      const double2 xv = __ldg(xr + p * W);
      acc[p].x = fma(a, xv.x, acc[p].x);
      acc[p].y = fma(a, xv.y, acc[p].y);
    }
  }
#pragma unroll
  for (int p = 0; p < TP; ++p) {
    if (ACC) {
      double2 o = yo[p];
      o.x += acc[p].x;
      o.y += acc[p].y;
      yr[p * W] = o;
    } else {
      yr[p * W] = acc[p];
    }
  }
}

// Small levels (few (row, time-pair) items): the S warps of a CTA share 32 consecutive items
// of one row (NT2 % 32 == 0) and split the row's entries (warp w: entries w, w + S, ...); the
// partial sums meet in shared memory.  Keeps every SM busy where one thread per item would fill
// a fraction of them (C2: restriction to levels 0 / 1 25 -> a few us).
template <bool ACC, int S>
__global__ void __launch_bounds__(32 * S) k_spmv_nt_split(int64_t nrow, int64_t NT2, const int32_t *__restrict__ rp,
                                                           const int32_t *__restrict__ ci,
                                                           const double *__restrict__ v,
                                                           const double2 *__restrict__ x, double2 *__restrict__ y) {
  __shared__ double2 part[S][32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t idx = blockIdx.x * 32ll + lane;  // the 32 items of a CTA lie in one row
  const int64_t i = (blockIdx.x * 32ll) / NT2, t = idx - i * NT2;
  const int e0 = __ldg(rp + i), e1 = __ldg(rp + i + 1);
  double2 acc = make_double2(0.0, 0.0);
#pragma unroll 4
  for (int e = e0 + w; e < e1; e += S) {
    const double a = __ldg(v + e);
    const double2 xv = __ldg(x + (int64_t)__ldg(ci + e) * NT2 + t);
    acc.x = fma(a, xv.x, acc.x);
    acc.y = fma(a, xv.y, acc.y);
  }
  part[w][lane] = acc;
  __syncthreads();
  if (w == 0) {
#pragma unroll
    for (int k = 1; k < S; ++k) {
      acc.x += part[k][lane].x;
      acc.y += part[k][lane].y;
    }
    if (ACC) {
      if (e0 == e1) return;
      double2 o = y[idx];
      o.x += acc.x;
      o.y += acc.y;
      y[idx] = o;
    } else {
      y[idx] = acc;
    }
  }
}

void spmv_nt(const DevCSR &A, int64_t NT, const double *x, double *y, bool acc, cudaStream_t s) {
  static const int tp = [] {  // WRMG_SPMV_TP=1: one time pair per thread (A/B)
    const char *e = getenv("WRMG_SPMV_TP");
    return e ? atoi(e) : 4;
  }();
  // launch shape by level size: four time pairs per thread only where the items still fill the
  // GPU twice over, one pair per thread in between, entry-split CTAs on the small levels
  const int64_t items = A.nrow * (NT / 2);
  const int64_t fill = (int64_t)num_sms() * 2048;
  if (NT % 2 == 0 && (NT / 2) % 32 == 0 && items < fill / 2 && tp != 1) {
    const unsigned nb = (unsigned)(items / 32);
    if (acc)
      k_spmv_nt_split<true, 8><<<nb, 256, 0, s>>>(A.nrow, NT / 2, A.rowptr, A.col, A.val, (const double2 *)x,
                                                   (double2 *)y);
    else
      k_spmv_nt_split<false, 8><<<nb, 256, 0, s>>>(A.nrow, NT / 2, A.rowptr, A.col, A.val, (const double2 *)x,
                                                    (double2 *)y);
    ++g_launches;
    return;
  }
  if (NT % 2 == 0 && tp == 4 && (NT / 2) % 4 == 0 && items / 4 >= fill / 3) {
    const int64_t n = A.nrow * (NT / 8);
    if (acc)
      k_spmv_nt_tp<true, 4><<<(unsigned)((n + 255) / 256), 256, 0, s>>>(A.nrow, NT / 2, A.rowptr, A.col, A.val,
                                                                         (const double2 *)x, (double2 *)y);
    else
      k_spmv_nt_tp<false, 4><<<(unsigned)((n + 255) / 256), 256, 0, s>>>(A.nrow, NT / 2, A.rowptr, A.col, A.val,
                                                                          (const double2 *)x, (double2 *)y);
    ++g_launches;
    return;
  }
  if (NT % 2 == 0) {
    const int64_t n = A.nrow * (NT / 2);
    if (acc)
      k_spmv_nt<true><<<(unsigned)((n + 255) / 256), 256, 0, s>>>(A.nrow, NT / 2, A.rowptr, A.col, A.val,
                                                                  (const double2 *)x, (double2 *)y);
    else
      k_spmv_nt<false><<<(unsigned)((n + 255) / 256), 256, 0, s>>>(A.nrow, NT / 2, A.rowptr, A.col, A.val,
                                                                   (const double2 *)x, (double2 *)y);
  } else {
    const int64_t n = A.nrow * NT;
    k_spmv_nt1<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(A.nrow, NT, A.rowptr, A.col, A.val, x, y, acc);
  }
  ++g_launches;
}

// ------------------------------------------------------------- coarse solve
// H11: exact block forward substitution over slabs for one "patch" holding all
// free coarse nodes: z_n = D^{-1} g_n (slab-parallel), y_n = z_n[q] + G_q y_{n-1}
// (one CTA, sequential), x_n = z_n + G y_{n-1} (slab-parallel).
__global__ void __launch_bounds__(256) k_coarse_z(int m, int mp, int nq, int64_t NT, const int32_t *__restrict__ nodes,
                                                  const double *__restrict__ DinvT, const double *__restrict__ r,
                                                  double *__restrict__ Z) {
  extern __shared__ double g[];
  const int n = blockIdx.x;
  for (int rho = threadIdx.x; rho < m; rho += blockDim.x) {
    int a = rho / mp, i = rho % mp;
    g[rho] = r[(int64_t)nodes[i] * NT + (int64_t)n * nq + a];
  }
  __syncthreads();
  for (int rho = threadIdx.x; rho < m; rho += blockDim.x) {
    double acc = 0.0;
    for (int sg = 0; sg < m; ++sg) acc = fma(DinvT[(int64_t)sg * m + rho], g[sg], acc);
    Z[(int64_t)n * m + rho] = acc;
  }
}

__global__ void __launch_bounds__(1024) k_coarse_rec(int N, int m, int mp, int nq, const double *__restrict__ Z,
                                                     const double *__restrict__ Gq, double *__restrict__ Y,
                                                     int gq_in_smem) {
  extern __shared__ double sg[];
  double *ysm = sg;             // 2 * mp
  double *gqs = sg + 2 * mp;    // mp * mp (optional)
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, nw = blockDim.x >> 5;
  if (gq_in_smem)
    for (int e = tid; e < mp * mp; e += blockDim.x) gqs[e] = Gq[e];
  for (int i = tid; i < mp; i += blockDim.x) {
    ysm[i] = 0.0;
    Y[i] = 0.0;
  }
  __syncthreads();
  const double *G = gq_in_smem ? gqs : Gq;
  for (int n = 0; n < N; ++n) {
    const double *yprev = ysm + (n & 1) * mp;
    double *ynew = ysm + ((n + 1) & 1) * mp;
    for (int i = wid; i < mp; i += nw) {
      double acc = 0.0;
      for (int j = lane; j < mp; j += 32) acc = fma(G[(int64_t)i * mp + j], yprev[j], acc);
      for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
      if (lane == 0) {
        double y = Z[(int64_t)n * m + (nq - 1) * mp + i] + acc;
        ynew[i] = y;
        Y[(int64_t)(n + 1) * mp + i] = y;
      }
    }
    __syncthreads();
  }
}

__global__ void __launch_bounds__(256) k_coarse_x(int m, int mp, int nq, int64_t NT, const int32_t *__restrict__ nodes,
                                                  const double *__restrict__ Z, const double *__restrict__ GT,
                                                  const double *__restrict__ Y, double *__restrict__ x) {
  const int n = blockIdx.x;
  const double *yp = Y + (int64_t)n * mp;
  for (int rho = threadIdx.x; rho < m; rho += blockDim.x) {
    int a = rho / mp, i = rho % mp;
    double v;
    if (a == nq - 1) {
      v = Y[(int64_t)(n + 1) * mp + i];
    } else {
      v = Z[(int64_t)n * m + rho];
      for (int j = 0; j < mp; ++j) v = fma(GT[(int64_t)j * m + rho], yp[j], v);
    }
    x[(int64_t)nodes[i] * NT + (int64_t)n * nq + a] = v;
  }
}

// ----------------------------------------------------------------------- RHS
// b = (M (x) I_N (x) Mt) fhat on free rows (R6), 0 on constrained rows.
template <int NQ>
__global__ void k_rhs(int64_t nnode, int N, const int32_t *__restrict__ rp, const int32_t *__restrict__ ci,
                      const double *__restrict__ Mv, const uint8_t *__restrict__ con, const double *__restrict__ f,
                      double *__restrict__ b, TMc tm) {
  int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (idx >= nnode * N) return;
  int64_t i = idx / N;
  int n = (int)(idx - i * N);
  const int64_t NT = (int64_t)N * NQ;
  double* dst = b + i * NT + (int64_t)n * NQ;
  if (con[i]) {
    for (int a = 0; a < NQ; ++a) dst[a] = 0.0;
    return;
  }
  double mf[NQ];
  for (int a = 0; a < NQ; ++a) mf[a] = 0.0;
  for (int e = rp[i]; e < rp[i + 1]; ++e) {
    const double *src = f + (int64_t)ci[e] * NT + (int64_t)n * NQ;
    for (int a = 0; a < NQ; ++a) mf[a] = fma(Mv[e], src[a], mf[a]);
  }
  for (int a = 0; a < NQ; ++a) {
    double acc = 0.0;
    for (int c = 0; c < NQ; ++c) acc = fma(tm.Mt[a * NQ + c], mf[c], acc);
    dst[a] = acc;
  }
}

// splitmix64 finaliser (R6), independent of wrmg_inputs.py.
__global__ void k_fill_uniform(double *out, int64_t count, unsigned long long first, unsigned long long seed) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= count) return;
  unsigned long long z = first + (unsigned long long)t + (seed + 1ull) * 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  z ^= z >> 31;
  out[t] = 2.0 * (double)(z >> 11) * 0x1.0p-53 - 1.0;
}

}  // namespace

void launch_residual(const Level &L, int q, int N, const Temporal &tm, const double *u, const double *b, double *r,
                     bool u_is_zero, cudaStream_t s) {
  const int64_t NT = (int64_t)N * (q + 1);
  if (u_is_zero) {
    if (b) cudaMemcpyAsync(r, b, L.nnode * NT * sizeof(double), cudaMemcpyDeviceToDevice, s);
    else cudaMemsetAsync(r, 0, L.nnode * NT * sizeof(double), s);
    return;
  }
  const int k = (L.Lx - 1) / L.nx;
  static const int64_t mac_min = [] {  // level size from which the macro-block residual runs
    const char *e = getenv("WRMG_MAC_MIN_NODES");
    return e ? (int64_t)atoll(e) : (int64_t)5000;  // C2: L3 (9409 nodes) 35 vs 44 us, L2 (2401) 29 vs 16 us
  }();
  if (L.nnode >= mac_min && launch_residual_mac(L, k, q, N, tm, u, b, r, s)) return;
  if (launch_residual_cls(L, q, N, tm, u, b, r, s)) return;
  const int ntx = (L.Lx + RT - 1) / RT, nty = (L.Ly + RT - 1) / RT;
  dim3 grid(ntx * nty, (N + RCS - 1) / RCS);
  const int RW = RT + 2 * k;
  size_t smem = (size_t)RW * RW * (RCS * (q + 1) + 1) * sizeof(double);
  TMc t = make_tmc(tm);
#define WRMG_RES(NQ)                                                                                            \
  {                                                                                                             \
    smem_optin((const void *)k_residual<NQ>, 200 * 1024);                                                                                                           \
    k_residual<NQ><<<grid, 256, smem, s>>>(k, L.Lx, L.Ly, N, L.A.rowptr, L.A.col, L.A.val, L.A.val2, L.con, u, b, \
                                           r, t); ++g_launches;                                                               \
  }
  switch (q) {
    case 0: WRMG_RES(1); break;
    case 1: WRMG_RES(2); break;
    case 2: WRMG_RES(3); break;
    default: WRMG_RES(4); break;
  }
#undef WRMG_RES
}

void launch_sweep(const Level &L, int q, int N, const double *r, double *u, double omega, cudaStream_t s) {
  const int nq = q + 1;
#define WRMG_SW(NQ, MP) \
  if (nq == NQ && L.mp == MP) return sweep_launch<NQ, MP>(L, N, r, u, omega, s);
  WRMG_SW(1, 1) WRMG_SW(2, 1) WRMG_SW(3, 1) WRMG_SW(4, 1)
  WRMG_SW(1, 7) WRMG_SW(2, 7) WRMG_SW(3, 7) WRMG_SW(4, 7)
  WRMG_SW(1, 19) WRMG_SW(2, 19) WRMG_SW(3, 19) WRMG_SW(4, 19)
#undef WRMG_SW
}

void launch_restrict(const Level &C, int64_t NT, const double *rf, double *rc, cudaStream_t s) {
  spmv_nt(C.R, NT, rf, rc, false, s);
}

void launch_prolong_add(const Level &C, int64_t NT, const double *ec, double *uf, cudaStream_t s) {
  spmv_nt(C.P, NT, ec, uf, true, s);
}

void launch_coarse_solve(const Coarse &C, const Level &L, int q, int N, const double *r, double *x, cudaStream_t s) {
  const int nq = q + 1;
  const int64_t NT = (int64_t)N * nq;
  cudaMemsetAsync(x, 0, L.nnode * NT * sizeof(double), s);
  smem_optin((const void *)k_coarse_z, C.m * (int)sizeof(double));
  k_coarse_z<<<N, 256, C.m * sizeof(double), s>>>(C.m, C.mp, nq, NT, C.nodes, C.DinvT, r, C.Z); ++g_launches;
  size_t gq = (size_t)C.mp * C.mp * sizeof(double);
  int in_smem = (gq + 2 * C.mp * sizeof(double)) <= 200 * 1024;
  size_t smem = 2 * C.mp * sizeof(double) + (in_smem ? gq : 0);
  smem_optin((const void *)k_coarse_rec, 210 * 1024);
  k_coarse_rec<<<1, 1024, smem, s>>>(N, C.m, C.mp, nq, C.Z, C.Gq, C.Y, in_smem); ++g_launches;
  k_coarse_x<<<N, 256, 0, s>>>(C.m, C.mp, nq, NT, C.nodes, C.Z, C.GT, C.Y, x); ++g_launches;
}

void launch_rhs(const Level &L, int q, int N, const Temporal &tm, const double *f, double *b, cudaStream_t s) {
  int64_t n = L.nnode * N;
  unsigned blocks = (unsigned)((n + 255) / 256);
  TMc t = make_tmc(tm);
  switch (q) {
    case 0: k_rhs<1><<<blocks, 256, 0, s>>>(L.nnode, N, L.A.rowptr, L.A.col, L.A.val, L.con, f, b, t); ++g_launches; break;
    case 1: k_rhs<2><<<blocks, 256, 0, s>>>(L.nnode, N, L.A.rowptr, L.A.col, L.A.val, L.con, f, b, t); ++g_launches; break;
    case 2: k_rhs<3><<<blocks, 256, 0, s>>>(L.nnode, N, L.A.rowptr, L.A.col, L.A.val, L.con, f, b, t); ++g_launches; break;
    default: k_rhs<4><<<blocks, 256, 0, s>>>(L.nnode, N, L.A.rowptr, L.A.col, L.A.val, L.con, f, b, t); ++g_launches; break;
  }
}

void launch_fill_uniform(double *out, int64_t count, uint64_t first, uint64_t seed, cudaStream_t s) {
  if (count <= 0) return;
  k_fill_uniform<<<(unsigned)((count + 255) / 256), 256, 0, s>>>(out, count, first, seed); ++g_launches;
}

}  // namespace wrmg
