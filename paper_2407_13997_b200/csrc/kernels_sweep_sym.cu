// Waveform-relaxation patch sweep (H7 + H8) for the interior vertex-star class
// in the symmetry-adapted Kronecker basis (host_sym.cu derives it):
//
//   g   = R_p r_n                       gather, slot order of host_sym.cu
//   y   = U^T g                         orbit sums / differences (adds only)
//   gh  = diag(V_chi)^T y               four small blocks: sum d_chi^2 FMAs (P3: 99, not 361)
//   per mode i: t = S_i gh_i, end trace y_{n,i} = t[q] + sigma_i y_{n-1,i} (scan over slabs),
//               w = t + S_i[:, 0] y_{n-1,i} (a < q),  w[q] = y_{n,i}       (kernels_kron.cu)
//   x   = U diag(V_chi) w
//   u  += omega W_p x                   FP64 atomics (weighted additive scatter, R11)
//
// Warp = one patch, lane = one slab of a 32-slab chunk holding its NQ values; the
// warp walks the chunks in order, the end-trace carry of every mode kept in shared
// memory; one character block at a time is live in registers besides y.  The
// block coefficients are kernel parameters (constant bank operands).  Patches of the
// other (boundary) classes go through kernels_kron.cu on their own work lists.
#include <cstdlib>

#include "internal.h"
#include "sym.h"

namespace wrmg {
namespace {

template <int K>
struct SymShape;
template <>
struct SymShape<2> {
  static constexpr int N1 = 1, N2 = 1, N3 = 0;
};
template <>
struct SymShape<3> {
  static constexpr int N1 = 3, N2 = 2, N3 = 1;
};

template <int K>
struct Sh {
  static constexpr int N1 = SymShape<K>::N1, N2 = SymShape<K>::N2, N3 = SymShape<K>::N3;
  static constexpr int MP = 1 + 4 * N1 + 2 * N2 + 2 * N3;
  static constexpr int D0 = 1 + N1 + N2 + N3, D1 = N1, D2 = N1 + N3, D3 = N1 + N2;
  static constexpr int B0 = 0, B1 = D0, B2 = D0 + D1, B3 = D0 + D1 + D2;
  static constexpr int V0 = 0, V1 = D0 * D0, V2 = V1 + D1 * D1, V3 = V2 + D2 * D2;
  static constexpr int T1 = 1, T2 = 1 + 4 * N1, T3 = 1 + 4 * N1 + 2 * N2;  // first slot of each orbit type
};

constexpr double kR = 0.70710678118654752440;  // 1/sqrt(2)
// Tile-interior nodes by plain read-modify-write: measured slower (each RMW waits on
// its load; 909 vs 428 us at C2 L5), so every union node goes through FP64 atomics
// (contiguous, 58 instead of 76 node updates per 2 x 2 tile at P3).
constexpr bool kTilePlainRMW = false;

// y = U^T g (slot order -> block coordinates)
template <int K>
__device__ __forceinline__ void sym_fwd(const double (&g)[Sh<K>::MP], double (&y)[Sh<K>::MP]) {
  using S = Sh<K>;
  y[S::B0] = g[0];
#pragma unroll
  for (int o = 0; o < S::N1; ++o) {
    const double x0 = g[S::T1 + 4 * o], x1 = g[S::T1 + 4 * o + 1], x2 = g[S::T1 + 4 * o + 2],
                 x3 = g[S::T1 + 4 * o + 3];
    const double s01 = x0 + x1, d01 = x0 - x1, s23 = x2 + x3, d23 = x2 - x3;
    y[S::B0 + 1 + o] = 0.5 * (s01 + s23);
    y[S::B1 + o] = 0.5 * (s01 - s23);
    y[S::B2 + o] = 0.5 * (d01 + d23);
    y[S::B3 + o] = 0.5 * (d01 - d23);
  }
#pragma unroll
  for (int o = 0; o < S::N2; ++o) {
    const double x0 = g[S::T2 + 2 * o], x1 = g[S::T2 + 2 * o + 1];
    y[S::B0 + 1 + S::N1 + o] = kR * (x0 + x1);
    y[S::B3 + S::N1 + o] = kR * (x0 - x1);
  }
#pragma unroll
  for (int o = 0; o < S::N3; ++o) {
    const double x0 = g[S::T3 + 2 * o], x1 = g[S::T3 + 2 * o + 1];
    y[S::B0 + 1 + S::N1 + S::N2 + o] = kR * (x0 + x1);
    y[S::B2 + S::N1 + o] = kR * (x0 - x1);
  }
}

// x = U y (block coordinates -> slot order)
template <int K>
__device__ __forceinline__ void sym_bwd(const double (&y)[Sh<K>::MP], double (&x)[Sh<K>::MP]) {
  using S = Sh<K>;
  x[0] = y[S::B0];
#pragma unroll
  for (int o = 0; o < S::N1; ++o) {
    const double a = y[S::B0 + 1 + o], b = y[S::B1 + o], c = y[S::B2 + o], d = y[S::B3 + o];
    const double ab = a + b, amb = a - b, cd = c + d, cmd = c - d;
    x[S::T1 + 4 * o] = 0.5 * (ab + cd);
    x[S::T1 + 4 * o + 1] = 0.5 * (ab - cd);
    x[S::T1 + 4 * o + 2] = 0.5 * (amb + cmd);
    x[S::T1 + 4 * o + 3] = 0.5 * (amb - cmd);
  }
#pragma unroll
  for (int o = 0; o < S::N2; ++o) {
    const double a = y[S::B0 + 1 + S::N1 + o], d = y[S::B3 + S::N1 + o];
    x[S::T2 + 2 * o] = kR * (a + d);
    x[S::T2 + 2 * o + 1] = kR * (a - d);
  }
#pragma unroll
  for (int o = 0; o < S::N3; ++o) {
    const double a = y[S::B0 + 1 + S::N1 + S::N2 + o], c = y[S::B2 + S::N1 + o];
    x[S::T3 + 2 * o] = kR * (a + c);
    x[S::T3 + 2 * o + 1] = kR * (a - c);
  }
}

// One character block of the transformed patch solve, for all NQ temporal nodes:
//   gh = V_chi^T y_chi;  per mode i of the block: t = S_i gh, end-trace scan, carry;
//   y_chi <- V_chi w   (in place: y_chi is dead once gh is formed)
template <int D, int B, int VO, int MODE0, int NQ, int MP>
__device__ __forceinline__ void sym_block(const SymTab &P, double (&y)[NQ][MP], double *ycar, int lane) {
  double t[NQ][D];
#pragma unroll
  for (int a = 0; a < NQ; ++a)
#pragma unroll
    for (int i = 0; i < D; ++i) {
      double s = 0.0;
#pragma unroll
      for (int j = 0; j < D; ++j) s = fma(P.V[VO + j * D + i], y[a][B + j], s);
      t[a][i] = s;
    }
#pragma unroll
  for (int i = 0; i < D; ++i) {
    const int md = MODE0 + i;
    double gh[NQ];
#pragma unroll
    for (int a = 0; a < NQ; ++a) gh[a] = t[a][i];
#pragma unroll
    for (int a = 0; a < NQ; ++a) {
      double s = 0.0;
#pragma unroll
      for (int b2 = 0; b2 < NQ; ++b2) s = fma(P.S[md * 16 + a * NQ + b2], gh[b2], s);
      t[a][i] = s;
    }
    const double sg = P.sig[md];
    double v = t[NQ - 1][i], pp = sg;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const double o = __shfl_up_sync(0xffffffffu, v, d);
      v = fma(lane >= d ? pp : 0.0, o, v);
      pp *= pp;
    }
    double pw = 1.0, bs = sg;  // sigma^(lane + 1)
#pragma unroll
    for (int bit = 0; bit < 6; ++bit) {
      pw *= (((lane + 1) >> bit) & 1) ? bs : 1.0;
      bs *= bs;
    }
    const double yc = ycar[md];
    const double yn = fma(pw, yc, v);
    double yp = __shfl_up_sync(0xffffffffu, yn, 1);
    if (lane == 0) yp = yc;
#pragma unroll
    for (int a = 0; a < NQ - 1; ++a) t[a][i] = fma(P.S[md * 16 + a * NQ + 0], yp, t[a][i]);
    t[NQ - 1][i] = yn;
    const double last = __shfl_sync(0xffffffffu, yn, 31);
    __syncwarp();
    if (lane == 0) ycar[md] = last;
  }
#pragma unroll
  for (int a = 0; a < NQ; ++a)
#pragma unroll
    for (int j = 0; j < D; ++j) {
      double s = 0.0;
#pragma unroll
      for (int i = 0; i < D; ++i) s = fma(P.V[VO + j * D + i], t[a][i], s);
      y[a][B + j] = s;
    }
}

// One patch x one 32-slab chunk: gather, y = U^T g, the four character blocks
// (end-trace carry in ycar), x = U y, handed to emit(a, x[slot]) one temporal node
// at a time (short live ranges).
template <int K, int NQ, class EMIT>
__device__ __forceinline__ void sym_patch_chunk(const SymTab &P, const int *snode, double *ycar, int n, bool valid,
                                                int64_t NT, const double *__restrict__ r, int lane,
                                                const EMIT &emit) {
  using S = Sh<K>;
  constexpr int MP = S::MP;
  double y[NQ][MP];
  {  // gather (slot order) and y = U^T g
    double g[NQ][MP];
#pragma unroll
    for (int j = 0; j < MP; ++j) {
      const double *src = r + (int64_t)snode[j] * NT + (int64_t)n * NQ;
      if constexpr (NQ == 2) {
        const double2 v = valid ? __ldg(reinterpret_cast<const double2 *>(src)) : make_double2(0.0, 0.0);
        g[0][j] = v.x;
        g[1][j] = v.y;
      } else {
#pragma unroll
        for (int a = 0; a < NQ; ++a) g[a][j] = valid ? __ldg(src + a) : 0.0;
      }
    }
#pragma unroll
    for (int a = 0; a < NQ; ++a) sym_fwd<K>(g[a], y[a]);
  }
  sym_block<S::D0, S::B0, S::V0, S::B0, NQ, MP>(P, y, ycar, lane);
  sym_block<S::D1, S::B1, S::V1, S::B1, NQ, MP>(P, y, ycar, lane);
  sym_block<S::D2, S::B2, S::V2, S::B2, NQ, MP>(P, y, ycar, lane);
  sym_block<S::D3, S::B3, S::V3, S::B3, NQ, MP>(P, y, ycar, lane);
#pragma unroll
  for (int a = 0; a < NQ; ++a) {
    double x[MP];
    sym_bwd<K>(y[a], x);
    emit(a, x);
  }
}

// The same chunk with y kept in the warp's shared-memory buffer buf[slot][lane][a]
// instead of registers (fewer live registers -> more warps per SM); on return buf
// holds the weighted corrections wt[slot] x[slot] for the contiguous atomics.
template <int D, int B, int VO, int MODE0, int NQ>
__device__ __forceinline__ void sym_block_s(const SymTab &P, const double *spw, double *yb, double *ycar, int lane) {
  auto Y = [&](int j, int a) -> double & { return yb[j * 32 * NQ + a]; };
  double t[NQ][D];
#pragma unroll
  for (int a = 0; a < NQ; ++a) {
    double yv[D];
#pragma unroll
    for (int j = 0; j < D; ++j) yv[j] = Y(B + j, a);
#pragma unroll
    for (int i = 0; i < D; ++i) {
      double s = 0.0;
#pragma unroll
      for (int j = 0; j < D; ++j) s = fma(P.V[VO + j * D + i], yv[j], s);
      t[a][i] = s;
    }
  }
#pragma unroll
  for (int i = 0; i < D; ++i) {
    const int md = MODE0 + i;
    double gh[NQ];
#pragma unroll
    for (int a = 0; a < NQ; ++a) gh[a] = t[a][i];
#pragma unroll
    for (int a = 0; a < NQ; ++a) {
      double s = 0.0;
#pragma unroll
      for (int b2 = 0; b2 < NQ; ++b2) s = fma(P.S[md * 16 + a * NQ + b2], gh[b2], s);
      t[a][i] = s;
    }
    // inclusive scan of the end-trace recurrence over the warp's 32 slabs: predicated
    // DFMAs with the constant-bank sig^(2^k) (lanes below the distance keep v exactly,
    // as fma(0, o, v) would), and sig^(lane + 1) from the CTA's table
    double v = t[NQ - 1][i];
#pragma unroll
    for (int k2 = 0; k2 < 5; ++k2) {
      const double o = __shfl_up_sync(0xffffffffu, v, 1 << k2);
      if (lane >= (1 << k2)) v = fma(P.sig2[k2][md], o, v);
    }
    const double pw = spw[md * 32 + lane];
    const double yc = ycar[md];
    const double yn = fma(pw, yc, v);
    double yp = __shfl_up_sync(0xffffffffu, yn, 1);
    if (lane == 0) yp = yc;
#pragma unroll
    for (int a = 0; a < NQ - 1; ++a) t[a][i] = fma(P.S[md * 16 + a * NQ + 0], yp, t[a][i]);
    t[NQ - 1][i] = yn;
    const double last = __shfl_sync(0xffffffffu, yn, 31);
    __syncwarp();
    if (lane == 0) ycar[md] = last;
  }
#pragma unroll
  for (int a = 0; a < NQ; ++a)
#pragma unroll
    for (int j = 0; j < D; ++j) {
      double s = 0.0;
#pragma unroll
      for (int i = 0; i < D; ++i) s = fma(P.V[VO + j * D + i], t[a][i], s);
      Y(B + j, a) = s;
    }
}

template <int K, int NQ>
__device__ __forceinline__ void sym_patch_chunk_s(const SymTab &P, const double *spw, const int *snode, const double *swt,
                                                  double *ycar,
                                                  int n, bool valid, int64_t NT, const double *__restrict__ r,
                                                  int lane, double *buf) {
  using S = Sh<K>;
  constexpr int MP = S::MP;
  double *yb = buf + lane * NQ;
  {  // gather (slot order), y = U^T g into the buffer
    double g[NQ][MP];
#pragma unroll
    for (int j = 0; j < MP; ++j) {
      const double *src = r + (int64_t)snode[j] * NT + (int64_t)n * NQ;
      if constexpr (NQ == 2) {
        const double2 v = valid ? __ldg(reinterpret_cast<const double2 *>(src)) : make_double2(0.0, 0.0);
        g[0][j] = v.x;
        g[1][j] = v.y;
      } else {
#pragma unroll
        for (int a = 0; a < NQ; ++a) g[a][j] = valid ? __ldg(src + a) : 0.0;
      }
    }
#pragma unroll
    for (int a = 0; a < NQ; ++a) {
      double y[MP];
      sym_fwd<K>(g[a], y);
#pragma unroll
      for (int j = 0; j < MP; ++j) yb[j * 32 * NQ + a] = y[j];
    }
  }
  sym_block_s<S::D0, S::B0, S::V0, S::B0, NQ>(P, spw, yb, ycar, lane);
  sym_block_s<S::D1, S::B1, S::V1, S::B1, NQ>(P, spw, yb, ycar, lane);
  sym_block_s<S::D2, S::B2, S::V2, S::B2, NQ>(P, spw, yb, ycar, lane);
  sym_block_s<S::D3, S::B3, S::V3, S::B3, NQ>(P, spw, yb, ycar, lane);
#pragma unroll
  for (int a = 0; a < NQ; ++a) {
    double y[MP], x[MP];
#pragma unroll
    for (int j = 0; j < MP; ++j) y[j] = yb[j * 32 * NQ + a];
    sym_bwd<K>(y, x);
#pragma unroll
    for (int j = 0; j < MP; ++j) yb[j * 32 * NQ + a] = swt[j] * x[j];
  }
}

// Chunk-parallel form of one character block (levels with few patches): the CTA's
// four warps hold four consecutive 32-slab chunks of ONE patch.  Each warp scans its
// chunk with zero carry-in, publishes the zero-carry end trace of every mode, and
// after one barrier forms its true carry-in from the group's carry and the earlier
// warps' end traces, y_in(w) = sigma^{32 w} ycar + sum_{w' < w} sigma^{32 (w - 1 - w')}
// z(w') (the end-trace recurrence y_n = z_n + sigma y_{n-1} is linear): the slab
// recurrence is solved in parallel over 128 slabs instead of one warp walking them.
template <int D, int B, int VO, int MODE0, int NQ, int MP>
__device__ __forceinline__ void sym_block_cp(const SymTab &P, double *yb, const double *ycar_in, double *ycar_out,
                                             double *zend, int lane, int w) {
  auto Y = [&](int j, int a) -> double & { return yb[j * 32 * NQ + a]; };
  double t[NQ][D], vv[D];
#pragma unroll
  for (int a = 0; a < NQ; ++a) {
    double yv[D];
#pragma unroll
    for (int j = 0; j < D; ++j) yv[j] = Y(B + j, a);
#pragma unroll
    for (int i = 0; i < D; ++i) {
      double s = 0.0;
#pragma unroll
      for (int j = 0; j < D; ++j) s = fma(P.V[VO + j * D + i], yv[j], s);
      t[a][i] = s;
    }
  }
#pragma unroll
  for (int i = 0; i < D; ++i) {
    const int md = MODE0 + i;
    double gh[NQ];
#pragma unroll
    for (int a = 0; a < NQ; ++a) gh[a] = t[a][i];
#pragma unroll
    for (int a = 0; a < NQ; ++a) {
      double s = 0.0;
#pragma unroll
      for (int b2 = 0; b2 < NQ; ++b2) s = fma(P.S[md * 16 + a * NQ + b2], gh[b2], s);
      t[a][i] = s;
    }
    double v = t[NQ - 1][i], pp = P.sig[md];
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const double o = __shfl_up_sync(0xffffffffu, v, d);
      v = fma(lane >= d ? pp : 0.0, o, v);
      pp *= pp;
    }
    vv[i] = v;
    const double last = __shfl_sync(0xffffffffu, v, 31);
    if (lane == 0) zend[w * MP + md] = last;
  }
  __syncthreads();
#pragma unroll
  for (int i = 0; i < D; ++i) {
    const int md = MODE0 + i;
    const double sg = P.sig[md];
    double s32 = sg;
#pragma unroll
    for (int b = 0; b < 5; ++b) s32 *= s32;
    double yin = ycar_in[md];
    for (int w2 = 0; w2 < w; ++w2) yin = fma(s32, yin, zend[w2 * MP + md]);
    double pw = 1.0, bs = sg;  // sigma^(lane + 1)
#pragma unroll
    for (int bit = 0; bit < 6; ++bit) {
      pw *= (((lane + 1) >> bit) & 1) ? bs : 1.0;
      bs *= bs;
    }
    const double yn = fma(pw, yin, vv[i]);
    double yp = __shfl_up_sync(0xffffffffu, yn, 1);
    if (lane == 0) yp = yin;
#pragma unroll
    for (int a = 0; a < NQ - 1; ++a) t[a][i] = fma(P.S[md * 16 + a * NQ + 0], yp, t[a][i]);
    t[NQ - 1][i] = yn;
    if (w == 3 && lane == 31) ycar_out[md] = yn;  // carry of the next group of four chunks
  }
#pragma unroll
  for (int a = 0; a < NQ; ++a)
#pragma unroll
    for (int j = 0; j < D; ++j) {
      double s = 0.0;
#pragma unroll
      for (int i = 0; i < D; ++i) s = fma(P.V[VO + j * D + i], t[a][i], s);
      Y(B + j, a) = s;
    }
}

template <int K, int NQ>
__device__ __forceinline__ void sym_patch_chunk_cp(const SymTab &P, const int *snode, const double *swt,
                                                   const double *ycar_in, double *ycar_out, double *zend, int n,
                                                   bool valid, int64_t NT, const double *__restrict__ r, int lane,
                                                   int w, double *buf) {
  using S = Sh<K>;
  constexpr int MP = S::MP;
  double *yb = buf + lane * NQ;
  {
    double g[NQ][MP];
#pragma unroll
    for (int j = 0; j < MP; ++j) {
      const double *src = r + (int64_t)snode[j] * NT + (int64_t)n * NQ;
      if constexpr (NQ == 2) {
        const double2 v = valid ? __ldg(reinterpret_cast<const double2 *>(src)) : make_double2(0.0, 0.0);
        g[0][j] = v.x;
        g[1][j] = v.y;
      } else {
#pragma unroll
        for (int a = 0; a < NQ; ++a) g[a][j] = valid ? __ldg(src + a) : 0.0;
      }
    }
#pragma unroll
    for (int a = 0; a < NQ; ++a) {
      double y[MP];
      sym_fwd<K>(g[a], y);
#pragma unroll
      for (int j = 0; j < MP; ++j) yb[j * 32 * NQ + a] = y[j];
    }
  }
  sym_block_cp<S::D0, S::B0, S::V0, S::B0, NQ, MP>(P, yb, ycar_in, ycar_out, zend, lane, w);
  sym_block_cp<S::D1, S::B1, S::V1, S::B1, NQ, MP>(P, yb, ycar_in, ycar_out, zend, lane, w);
  sym_block_cp<S::D2, S::B2, S::V2, S::B2, NQ, MP>(P, yb, ycar_in, ycar_out, zend, lane, w);
  sym_block_cp<S::D3, S::B3, S::V3, S::B3, NQ, MP>(P, yb, ycar_in, ycar_out, zend, lane, w);
#pragma unroll
  for (int a = 0; a < NQ; ++a) {
    double y[MP], x[MP];
#pragma unroll
    for (int j = 0; j < MP; ++j) y[j] = yb[j * 32 * NQ + a];
    sym_bwd<K>(y, x);
#pragma unroll
    for (int j = 0; j < MP; ++j) yb[j * 32 * NQ + a] = swt[j] * x[j];
  }
}

// CTA = one patch, warp = one 32-slab chunk of a group of four (sym_block_cp).
template <int K, int NQ>
__global__ void __launch_bounds__(128, 4) k_sweep_sym_cp(int N, int64_t npatch, const int32_t *__restrict__ list,
                                                         const int32_t *__restrict__ pnodes,
                                                         const __grid_constant__ SymTab P,
                                                         const double *__restrict__ wnode, double omega,
                                                         const double *__restrict__ r, double *__restrict__ u) {
  constexpr int MP = Sh<K>::MP;
  __shared__ int snode[MP];
  __shared__ double swt[MP];
  __shared__ double sycar[2][MP];
  __shared__ double zend[4 * MP];
  extern __shared__ __align__(16) double stage[];  // [4][MP][32][NQ]
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t NT = (int64_t)N * NQ;
  const int nch = (N + 31) / 32, ngrp = (nch + 3) / 4;
  double *stg = stage + (size_t)w * MP * 32 * NQ;
  for (int64_t i = blockIdx.x; i < npatch; i += gridDim.x) {
    const int64_t p = list ? list[i] : i;
    __syncthreads();
    if (threadIdx.x < MP) {
      const int nd = __ldg(pnodes + p * MP + threadIdx.x);
      snode[threadIdx.x] = nd;
      swt[threadIdx.x] = omega * __ldg(wnode + nd);
      sycar[0][threadIdx.x] = 0.0;
    }
    __syncthreads();
    for (int g = 0; g < ngrp; ++g) {
      const int ch = 4 * g + w;
      const int n = 32 * ch + lane;
      sym_patch_chunk_cp<K, NQ>(P, snode, swt, sycar[g & 1], sycar[(g & 1) ^ 1], zend, n, n < N, NT, r, lane, w,
                                stg);
      __syncwarp();
      if (ch < nch) {
        const int64_t t0 = (int64_t)ch * 32 * NQ;
        const int nv = (int)min((int64_t)32 * NQ, NT - t0);
#pragma unroll 4
        for (int j = 0; j < MP; ++j) {
          double *dst = u + (int64_t)snode[j] * NT + t0;
#pragma unroll
          for (int e = 0; e < NQ; ++e) {
            const int idx = lane + 32 * e;
            if (idx < nv) atomicAdd(dst + idx, stg[j * 32 * NQ + idx]);
          }
        }
      }
      __syncthreads();  // the next group's carry is written; zend / stage reusable
    }
  }
}

// Chunk-parallel form: opt-in (WRMG_SWEEP_CP=1).
bool use_chunk_parallel(int64_t np, int N) {
  static const int mode = [] {
    const char *e = getenv("WRMG_SWEEP_CP");
    return e ? (e[0] == '1' ? 1 : 0) : -1;
  }();
  (void)np;
  return N > 32 && mode == 1;  // measured slower than one warp per patch at C2's 64^2 level
}

// Patches one per warp, FP64 atomics for the weighted additive scatter.
template <int K, int NQ>
__global__ void __launch_bounds__(128, 4) k_sweep_sym(int N, int64_t npatch, const int32_t *__restrict__ list,
                                                      const int32_t *__restrict__ pnodes,
                                                      const __grid_constant__ SymTab P,
                                                      const double *__restrict__ wnode, double omega,
                                                      const double *__restrict__ r, double *__restrict__ u) {
  constexpr int MP = Sh<K>::MP;
  constexpr int WPC = 4;
  __shared__ int snode[WPC][MP];
  __shared__ double swt[WPC][MP];
  __shared__ double sycar[WPC][MP];  // end trace of every mode at the previous chunk's last slab
  __shared__ double spw[MP * 32];     // sig_mode^(lane + 1): the carry's weight in the scan
  extern __shared__ __align__(16) double stage[];  // [WPC][MP][32][NQ]
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t NT = (int64_t)N * NQ;
  const int nch = (N + 31) / 32;
  for (int e = threadIdx.x; e < MP * 32; e += blockDim.x) {
    const int l = e & 31;
    double pw = 1.0, bs = P.sig[e >> 5];  // binary powering, as the in-warp form formed it
    for (int bit = 0; bit < 6; ++bit) {
      pw *= (((l + 1) >> bit) & 1) ? bs : 1.0;
      bs *= bs;
    }
    spw[e] = pw;
  }
  __syncthreads();
  for (int64_t i = (int64_t)blockIdx.x * WPC + w; i < npatch; i += (int64_t)gridDim.x * WPC) {
    const int64_t p = list ? list[i] : i;
    __syncwarp();
    if (lane < MP) {
      const int nd = __ldg(pnodes + p * MP + lane);
      snode[w][lane] = nd;
      swt[w][lane] = omega * __ldg(wnode + nd);
      sycar[w][lane] = 0.0;
    }
    __syncwarp();
    for (int ch = 0; ch < nch; ++ch) {
      const int n = 32 * ch + lane;
      const bool valid = n < N;
      // stage the weighted corrections [slot][slab][a] in shared memory, then one
      // contiguous run of 32 NQ atomics per node (lanes on consecutive doubles: fewer
      // L2 sectors per instruction than lane = slab with stride NQ)
      double *stg = stage + (size_t)w * MP * 32 * NQ;
      sym_patch_chunk_s<K, NQ>(P, spw, snode[w], swt[w], sycar[w], n, valid, NT, r, lane, stg);
      __syncwarp();
      const int64_t t0 = (int64_t)ch * 32 * NQ;
      const int nv = (int)min((int64_t)32 * NQ, NT - t0);  // valid values of this chunk
#pragma unroll 4
      for (int j = 0; j < MP; ++j) {
        double *dst = u + (int64_t)snode[w][j] * NT + t0;
#pragma unroll
        for (int e = 0; e < NQ; ++e) {
          const int idx = lane + 32 * e;
          if (idx < nv) atomicAdd(dst + idx, stg[j * 32 * NQ + idx]);
        }
      }
      __syncwarp();
    }
  }
}

// 2 x 2 vertex tiles (CTA = 4 warps = 4 patches): the patches' corrections meet in
// shared memory, each union node of the tile is written once per chunk as 32 NQ
// contiguous doubles -- plain read-modify-write for nodes no other tile touches,
// FP64 atomics for the tile's boundary nodes (k = 3: 42 atomic + 16 plain node
// updates instead of 76 atomic ones).
template <int K, int NQ>
__global__ void __launch_bounds__(128, 3) k_sweep_sym_tile(int N, int64_t ntile, const int32_t *__restrict__ tiles,
                                                           const int32_t *__restrict__ pnodes,
                                                           const __grid_constant__ SymTab P,
                                                           const TileGeom *__restrict__ Tg,
                                                           const double *__restrict__ wnode, double omega,
                                                           const double *__restrict__ r, double *__restrict__ u) {
  constexpr int MP = Sh<K>::MP;
  constexpr int VC = 32 * NQ;  // doubles per node and chunk
  __shared__ int snode[4][MP];
  __shared__ double sycar[4][MP];
  __shared__ int32_t toff[kTileMaxU];
  __shared__ int16_t tsrc[kTileMaxU][4];
  __shared__ uint8_t tcnt[kTileMaxU], tint[kTileMaxU];
  extern __shared__ __align__(16) double acc_dyn[];  // [4][MP][VC]
  double(*acc)[MP][VC] = reinterpret_cast<double(*)[MP][VC]>(acc_dyn);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t NT = (int64_t)N * NQ;
  const int nch = (N + 31) / 32;
  const int nu = Tg->nu;
  for (int e = threadIdx.x; e < nu; e += blockDim.x) {  // tile geometry into shared memory
    toff[e] = Tg->off[e];
    tcnt[e] = Tg->cnt[e];
    tint[e] = Tg->interior[e];
    for (int q = 0; q < 4; ++q) tsrc[e][q] = Tg->src[e][q];
  }
  for (int64_t tl = blockIdx.x; tl < ntile; tl += gridDim.x) {
    __syncthreads();
    const int64_t p = tiles[tl * 4 + w];
    if (lane < MP) {
      snode[w][lane] = __ldg(pnodes + p * MP + lane);
      sycar[w][lane] = 0.0;
    }
    __syncthreads();
    // tile base node: the node of union offset 0 relative position, from patch 0's first slot
    const int64_t base = (int64_t)snode[0][tsrc[0][0] % MP] - toff[0];
    for (int ch = 0; ch < nch; ++ch) {
      const int n = 32 * ch + lane;
      const bool valid = n < N;
      sym_patch_chunk<K, NQ>(P, snode[w], sycar[w], n, valid, NT, r, lane, [&](int a, const double(&x)[MP]) {
#pragma unroll
        for (int j = 0; j < MP; ++j) acc[w][j][lane * NQ + a] = x[j];
      });
      __syncthreads();
      const int64_t t0 = (int64_t)ch * VC;  // first time value of the chunk
      for (int uu = w; uu < nu; uu += 4) {
        const int64_t node = base + toff[uu];
        const double wt = omega * __ldg(wnode + node);
        const int cnt = tcnt[uu];
        const bool inner = tint[uu];
        double *dst = u + node * NT + t0;
#pragma unroll
        for (int e = 0; e < NQ; ++e) {
          const int idx = lane + 32 * e;
          double v = 0.0;
          for (int q = 0; q < cnt; ++q) {
            const int sw = tsrc[uu][q];
            v += acc[sw / MP][sw % MP][idx];
          }
          if (t0 + idx < NT) {
            if (inner && kTilePlainRMW) dst[idx] += wt * v;
            else atomicAdd(dst + idx, wt * v);  // fire-and-forget: no load latency in the loop
          }
        }
      }
      __syncthreads();
    }
  }
}

template <int K, int NQ>
void sym_launch(const Level &L, int N, const double *r, double *u, double omega, cudaStream_t s) {
  if (L.ntile > 0) {
    const int grid = (int)std::min<int64_t>(L.ntile, (int64_t)6 * num_sms());
    const int smem = 4 * Sh<K>::MP * 32 * NQ * (int)sizeof(double);
    smem_optin((const void *)k_sweep_sym_tile<K, NQ>, smem);
    k_sweep_sym_tile<K, NQ><<<grid, 128, smem, s>>>(N, L.ntile, L.tile_patch, L.sym_nodes, L.symtab, L.tgeo_dev, L.wnode,
                                                  omega, r, u);
    ++g_launches;
  }
  const int64_t np = L.ntile > 0 ? L.nsingle : L.nsym;
  if (np > 0 && use_chunk_parallel(np, N)) {
    const int grid = (int)std::min<int64_t>(np, (int64_t)16 * num_sms());
    const int smem = 4 * Sh<K>::MP * 32 * NQ * (int)sizeof(double);
    smem_optin((const void *)k_sweep_sym_cp<K, NQ>, smem);
    k_sweep_sym_cp<K, NQ><<<grid, 128, smem, s>>>(N, np, L.ntile > 0 ? L.sym_single : nullptr, L.sym_nodes,
                                                  L.symtab, L.wnode, omega, r, u);
    ++g_launches;
  } else if (np > 0) {
    const int64_t nblk = (np + 3) / 4;
    const int grid = (int)std::min<int64_t>(nblk, (int64_t)10 * num_sms());
    const int smem = 4 * Sh<K>::MP * 32 * NQ * (int)sizeof(double);
    smem_optin((const void *)k_sweep_sym<K, NQ>, smem);
    k_sweep_sym<K, NQ><<<grid, 128, smem, s>>>(N, np, L.ntile > 0 ? L.sym_single : nullptr, L.sym_nodes, L.symtab,
                                               L.wnode, omega, r, u);
    ++g_launches;
  }
}

template <int K, int NQ>
void sym_list_launch(const Level &L, int N, const double *r, double *u, double omega, cudaStream_t s, int64_t np,
                     const int32_t *list) {
  if (np <= 0) return;
  const int smem = 4 * Sh<K>::MP * 32 * NQ * (int)sizeof(double);
  if (use_chunk_parallel(np, N)) {
    smem_optin((const void *)k_sweep_sym_cp<K, NQ>, smem);
    k_sweep_sym_cp<K, NQ><<<(int)std::min<int64_t>(np, (int64_t)16 * num_sms()), 128, smem, s>>>(
        N, np, list, L.sym_nodes, L.symtab, L.wnode, omega, r, u);
    ++g_launches;
    return;
  }
  const int grid = (int)std::min<int64_t>((np + 3) / 4, (int64_t)10 * num_sms());
  smem_optin((const void *)k_sweep_sym<K, NQ>, smem);
  k_sweep_sym<K, NQ><<<grid, 128, smem, s>>>(N, np, list, L.sym_nodes, L.symtab, L.wnode, omega, r, u);
  ++g_launches;
}

}  // namespace

bool launch_sweep_sym(const Level &L, int k, int q, int N, const double *r, double *u, double omega,
                      cudaStream_t s, const SweepLists *sl) {
  if (!L.sym_ok || L.nsym == 0) return false;
#define WRMG_SYM(KK_, NQ_)                                                            \
  if (k == KK_ && q + 1 == NQ_) {                                                     \
    if (sl) sym_list_launch<KK_, NQ_>(L, N, r, u, omega, s, sl->nsym, sl->sym_list); \
    else sym_launch<KK_, NQ_>(L, N, r, u, omega, s);                                 \
    return true;                                                                      \
  }
  WRMG_SYM(2, 1) WRMG_SYM(2, 2) WRMG_SYM(2, 3) WRMG_SYM(2, 4)
  WRMG_SYM(3, 1) WRMG_SYM(3, 2) WRMG_SYM(3, 3)
#undef WRMG_SYM
  return false;
}

}  // namespace wrmg
