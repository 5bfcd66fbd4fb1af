// Space-time residual (H6), macro-block form:
//
//   r_n = b_n - [(C+E0) (x) M + Mt (x) kappa K] u_n + (E1 (x) M) u_{n-1}     (eq. heatfem, R1-R3)
//   constrained rows: r = b - u                                               (R5)
//
// On the anti-diagonal P_k lattice every interior row of the
// same type (I mod k, J mod k) has the same stencil.  A warp owns one macro
// block -- the k x k rows (k i + a, k j + b) -- for a chunk of VPC = NQ floor(32/NQ)
// consecutive time values (lane = one (slab, temporal node) value).  The k^2 rows
// touch only 7 / 22 / 43 distinct nodes (P1 / P2 / P3) against 7 / 46 / 153
// stencil entries, so each neighbour value is read from shared memory once and
// feeds every row that uses it (the unrolled code of residual_mac_gen.h); the
// mass and stiffness coefficients are kernel parameters (constant bank operands
// of the DFMAs), so the inner loop reads nothing but u.
//
// Staging: a CTA owns a strip of MX macro columns and a segment of JS macro rows
// and walks time chunks (outer) and macro rows (inner).  u arrives in groups of k
// node lines x (k MX + 2k) nodes x VPC values, one 3-D TMA box each (out-of-lattice
// halo zero-filled), through a ring of R groups with one mbarrier per slot; the
// producer thread keeps the ring one macro row ahead.  Macro row j needs the three
// groups j-1, j, j+1, so every u line is loaded once per (strip, chunk) apart from
// the strip's x halo and the segment's two halo groups.
//
// The DG(q) combination needs all NQ values of a slab: lane (n, a) gathers the
// row's (M u)_n[c] and (K u)_n[c] of its slab by shuffles; the upwind jump (M u)_{n-1}[q]
// is lane - 1's value (lane 0: the previous chunk's, kept per row in shared memory).
// Rows whose class is not the interior one of their type (Neumann boundaries,
// strip-local lattice edges) are recomputed after this kernel by k_residual_rows.
#include <cuda.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <string>

#include "internal.h"

namespace wrmg {
// value types of the L1 macro kernel (NQ doubles per lane) and their FMA, declared
// before the generated accumulation code that calls vfma
struct V3 {
  double x, y, z;
};
struct V4 {
  double2 a, b;
};
__device__ __forceinline__ void vfma(double &acc, double c, const double &v) { acc = fma(c, v, acc); }
__device__ __forceinline__ void vfma(double2 &acc, double c, const double2 &v) {
  acc.x = fma(c, v.x, acc.x);
  acc.y = fma(c, v.y, acc.y);
}
__device__ __forceinline__ void vfma(V3 &acc, double c, const V3 &v) {
  acc.x = fma(c, v.x, acc.x);
  acc.y = fma(c, v.y, acc.y);
  acc.z = fma(c, v.z, acc.z);
}
__device__ __forceinline__ void vfma(V4 &acc, double c, const V4 &v) {
  vfma(acc.a, c, v.a);
  vfma(acc.b, c, v.b);
}

}  // namespace wrmg

#include "residual_mac_gen.h"

namespace wrmg {
namespace {

struct MacArgs {
  MacCoef C;
  double CE[16], Mt[16];
};

__device__ __forceinline__ void mbar_init(uint64_t *bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"((unsigned)__cvta_generic_to_shared(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(
                   (unsigned)__cvta_generic_to_shared(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, unsigned parity) {
  const unsigned a = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(a),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_3d(void *dst, const CUtensorMap *map, int c0, int c1, int c2, uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
      "[%5];\n" ::"r"((unsigned)__cvta_generic_to_shared(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"((unsigned)__cvta_generic_to_shared(bar))
      : "memory");
}

template <int K, int VPC, int RWX>
__device__ __forceinline__ void mac_accum(const double *g0, const double *g1, const double *g2, const MacCoef &C,
                                          double (&am)[K * K], double (&ak)[K * K]) {
  if constexpr (K == 1) mac_accum_k1<RWX, VPC>(g0, g1, g2, C, am, ak);
  else if constexpr (K == 2) mac_accum_k2<RWX, VPC>(g0, g1, g2, C, am, ak);
  else mac_accum_k3<RWX, VPC>(g0, g1, g2, C, am, ak);
}

// Rows that are not interior-class (boundary rows with truncated stencils, strip-local
// lattice edges): warp = one listed row x 32 slabs, neighbour values through L1
// (the class tables of StencilTab, global element offsets goff).
template <int NQ>
__global__ void __launch_bounds__(256) k_residual_rows(int64_t nrows, const int32_t *__restrict__ rows, int N,
                                                       const uint8_t *__restrict__ rcls, const double *__restrict__ u,
                                                       const double *__restrict__ b, double *__restrict__ r,
                                                       MacArgs P, const StencilTab T,
                                                       const int64_t *__restrict__ goff, int apply) {
  const int64_t NT = (int64_t)N * NQ;
  const int lane = threadIdx.x & 31;
  const int64_t wg = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nchunk = (N + 31) / 32;
  if (wg >= nrows * nchunk) return;
  const int64_t i = rows[wg / nchunk];
  const int n = (int)(wg % nchunk) * 32 + lane;
  const bool valid = n < N;
  const int ns = valid ? n : N - 1;
  const int64_t base = i * NT + (int64_t)ns * NQ;
  const int cls = __ldg(rcls + i);
  double am[NQ], ak[NQ], ap = 0.0;
#pragma unroll
  for (int a = 0; a < NQ; ++a) am[a] = ak[a] = 0.0;
  const double *ub = u + base;
  const int64_t *go = goff + cls * kStencilMaxE;
  for (int e = 0; e < T.cnt[cls]; ++e) {
    const double *ul = ub + __ldg(go + e);
    const double mv = T.m[cls][e], kv = T.kk[cls][e];
#pragma unroll
    for (int a = 0; a < NQ; ++a) {
      const double x = __ldg(ul + a);
      am[a] = fma(mv, x, am[a]);
      ak[a] = fma(kv, x, ak[a]);
    }
    if (lane == 0 && n > 0) ap = fma(mv, __ldg(ul - 1), ap);
  }
  double jm = __shfl_up_sync(0xffffffffu, am[NQ - 1], 1);
  if (lane == 0) jm = ap;
  if (valid) {
#pragma unroll
    for (int a = 0; a < NQ; ++a) {
      double acc = apply ? 0.0 : __ldg(b + base + a);
#pragma unroll
      for (int c = 0; c < NQ; ++c) acc -= P.CE[a * NQ + c] * am[c] + P.Mt[a * NQ + c] * ak[c];
      if (a == 0 && n > 0) acc += jm;
      r[base + a] = apply ? -acc : acc;
    }
  }
}

// ---- L1 form: no staging.  Warp = one macro block x 32 slabs (lane = slab, its NQ
// values in registers: one vector load per union node and lane, every coefficient
// feeds NQ FMAs, the DG(q) combination is lane-local); the warp walks the 32-slab
// chunks of its macro in order, the jump carry (M u)_{last slab}[q] of every row in
// registers.  Neighbour values come through L1: the warps of a CTA take adjacent
// macros, so the halo lines they share are read once per SM.
template <int NQ>
struct VT;
template <>
struct VT<1> {
  using T = double;
  static __device__ __forceinline__ T ld(const double *p) { return __ldg(p); }
  static __device__ __forceinline__ T zero() { return 0.0; }
  static __device__ __forceinline__ double get(const T &v, int) { return v; }
  static __device__ __forceinline__ void st(double *p, const double (&o)[1]) { *p = o[0]; }
};
template <>
struct VT<2> {
  using T = double2;
  static __device__ __forceinline__ T ld(const double *p) { return __ldg(reinterpret_cast<const double2 *>(p)); }
  static __device__ __forceinline__ T zero() { return make_double2(0.0, 0.0); }
  static __device__ __forceinline__ double get(const T &v, int a) { return a ? v.y : v.x; }
  static __device__ __forceinline__ void st(double *p, const double (&o)[2]) {
    *reinterpret_cast<double2 *>(p) = make_double2(o[0], o[1]);
  }
};
template <>
struct VT<3> {
  using T = V3;
  static __device__ __forceinline__ T ld(const double *p) { return V3{__ldg(p), __ldg(p + 1), __ldg(p + 2)}; }
  static __device__ __forceinline__ T zero() { return V3{0.0, 0.0, 0.0}; }
  static __device__ __forceinline__ double get(const T &v, int a) { return a == 0 ? v.x : a == 1 ? v.y : v.z; }
  static __device__ __forceinline__ void st(double *p, const double (&o)[3]) {
    p[0] = o[0];
    p[1] = o[1];
    p[2] = o[2];
  }
};
template <>
struct VT<4> {
  using T = V4;
  static __device__ __forceinline__ T ld(const double *p) {
    return V4{__ldg(reinterpret_cast<const double2 *>(p)), __ldg(reinterpret_cast<const double2 *>(p + 2))};
  }
  static __device__ __forceinline__ T zero() { return V4{make_double2(0.0, 0.0), make_double2(0.0, 0.0)}; }
  static __device__ __forceinline__ double get(const T &v, int a) {
    return a == 0 ? v.a.x : a == 1 ? v.a.y : a == 2 ? v.b.x : v.b.y;
  }
  static __device__ __forceinline__ void st(double *p, const double (&o)[4]) {
    *reinterpret_cast<double2 *>(p) = make_double2(o[0], o[1]);
    *reinterpret_cast<double2 *>(p + 2) = make_double2(o[2], o[3]);
  }
};
// rows of macro line b = 0 (part 0) or b >= 1 (part 1); K = 1 has a single part
template <int K, class LD, class V>
__device__ __forceinline__ void mac_accum_ld_part(int part, const LD &ld, const MacCoef &C, V (&am)[K * K],
                                                  V (&ak)[K * K]) {
  if constexpr (K == 1) mac_accum_ld_k1(ld, C, am, ak);
  else if constexpr (K == 2) {
    if (part == 0) mac_accum_ld_k2_p0(ld, C, am, ak);
    else if (part == 1) mac_accum_ld_k2_p1(ld, C, am, ak);
    else mac_accum_ld_k2(ld, C, am, ak);
  } else {
    if (part == 0) mac_accum_ld_k3_p0(ld, C, am, ak);
    else if (part == 1) mac_accum_ld_k3_p1(ld, C, am, ak);
    else mac_accum_ld_k3(ld, C, am, ak);
  }
}

template <int K, class LD, class V>
__device__ __forceinline__ void mac_accum_ld(const LD &ld, const MacCoef &C, V (&am)[K * K], V (&ak)[K * K]) {
  if constexpr (K == 1) mac_accum_ld_k1(ld, C, am, ak);
  else if constexpr (K == 2) mac_accum_ld_k2(ld, C, am, ak);
  else mac_accum_ld_k3(ld, C, am, ak);
}

// one macro block, all time chunks; GUARD: the 3k x 3k window leaves the lattice
template <int K, int NQ, bool GUARD>
__device__ __forceinline__ void mac_l1_block(const MacArgs &P, int Lx, int Ly, int N, int X0, int Y0, int rc,
                                             const double *__restrict__ u, const double *__restrict__ b,
                                             double *__restrict__ r, int apply, int lane) {
  using W = VT<NQ>;
  using V = typename W::T;
  constexpr int KK = K * K;
  const int64_t NT = (int64_t)N * NQ;
  const int64_t LxNT = (int64_t)Lx * NT;
  const int nch = (N + 31) / 32;
  double prev[KK];
#pragma unroll
  for (int t = 0; t < KK; ++t) prev[t] = 0.0;
  // window origin (X0 - K, Y0 - K); window node (yl, xl) at element offset yl Lx NT + xl NT
  const double *wbase = u + (int64_t)(Y0 - K) * LxNT + (int64_t)(X0 - K) * NT;
  for (int c = 0; c < nch; ++c) {
    const int n = 32 * c + lane;
    const bool valid = n < N;
    const int64_t so = (int64_t)(valid ? n : N - 1) * NQ;
    const double *wl = wbase + so;
    auto ld = [&](int yl, int xl) -> V {
      if (GUARD) {
        const int X = X0 - K + xl, Y = Y0 - K + yl;
        if (X < 0 || Y < 0 || X >= Lx || Y >= Ly) return W::zero();
      }
      return W::ld(wl + (yl * LxNT + xl * NT));
    };
    V am[KK], ak[KK];
#pragma unroll
    for (int t = 0; t < KK; ++t) am[t] = ak[t] = W::zero();
    mac_accum_ld<K>(ld, P.C, am, ak);
#pragma unroll
    for (int t = 0; t < KK; ++t) {
      const int cls = __shfl_sync(0xffffffffu, rc, t);
      const double lastq = W::get(am[t], NQ - 1);
      double jmv = __shfl_up_sync(0xffffffffu, lastq, 1);
      if (lane == 0) jmv = prev[t];
      prev[t] = __shfl_sync(0xffffffffu, lastq, 31);
      const int64_t ro = (int64_t)(Y0 + t / K) * LxNT + (int64_t)(X0 + t % K) * NT + so;
      const bool inl = cls <= 0xFF;  // the row exists (partial macros at the far lattice edges)
      const V bv = (apply || !inl) ? W::zero() : W::ld(b + ro);
      double o[NQ];
#pragma unroll
      for (int a = 0; a < NQ; ++a) {
        double acc = W::get(bv, a);
#pragma unroll
        for (int c2 = 0; c2 < NQ; ++c2)
          acc -= P.CE[a * NQ + c2] * W::get(am[t], c2) + P.Mt[a * NQ + c2] * W::get(ak[t], c2);
        if (a == 0 && n > 0) acc += jmv;
        o[a] = apply ? -acc : acc;
      }
      if (cls == 0xFF) {  // constrained row: identity
        const V own = W::ld(u + ro);
#pragma unroll
        for (int a = 0; a < NQ; ++a) o[a] = apply ? W::get(own, a) : W::get(bv, a) - W::get(own, a);
      }
      if (valid && inl) W::st(r + ro, o);
    }
  }
}

template <int K, int NQ>
__global__ void __launch_bounds__(128, K == 3 ? 3 : 4) k_residual_mac_l1(const __grid_constant__ MacArgs P, int Lx,
                                                                         int Ly, int N, int nmx, int64_t nmac,
                                                                         const uint8_t *__restrict__ rcls,
                                                                         const double *__restrict__ u,
                                                                         const double *__restrict__ b,
                                                                         double *__restrict__ r, int apply) {
  constexpr int KK = K * K;
  const int lane = threadIdx.x & 31;
  const int64_t w0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t mi = w0; mi < nmac; mi += nw) {
    const int im = (int)(mi % nmx), jm = (int)(mi / nmx);
    const int X0 = K * im, Y0 = K * jm;
    int rc = 0x100;
    if (lane < KK) {
      const int X = X0 + lane % K, Y = Y0 + lane / K;
      if (X < Lx && Y < Ly) rc = __ldg(rcls + (int64_t)Y * Lx + X);
    }
    if (X0 < K || Y0 < K || X0 + 2 * K > Lx || Y0 + 2 * K > Ly)
      mac_l1_block<K, NQ, true>(P, Lx, Ly, N, X0, Y0, rc, u, b, r, apply, lane);
    else
      mac_l1_block<K, NQ, false>(P, Lx, Ly, N, X0, Y0, rc, u, b, r, apply, lane);
  }
}

template <int K, int NQ>
bool mac_l1_launch(const Level &L, int N, const MacArgs &P, const double *u, const double *b, double *r, int apply,
                   cudaStream_t s) {
  const int nmx = (L.Lx + K - 1) / K, nmy = (L.Ly + K - 1) / K;
  const int64_t nmac = (int64_t)nmx * nmy;
  const int64_t blocks = (nmac + 3) / 4;
  const int grid = (int)std::min<int64_t>(blocks, (int64_t)(K == 3 ? 3 : 4) * num_sms());
  k_residual_mac_l1<K, NQ><<<grid, 128, 0, s>>>(P, L.Lx, L.Ly, N, nmx, nmac, L.rcls, u, b, r, apply);
  ++g_launches;
  return true;
}

// ---- TMA form.  Warp = two adjacent macro blocks x 16 slabs (lane = (macro h, slab):
// half-warp h, its NQ values in registers); CTA = MX macro columns x JS macro rows,
// walking 16-slab chunks (outer) and macro rows (inner); u arrives in groups of k
// node lines x (k MX + 2k) nodes x 16 slabs through a ring of R TMA boxes (one
// mbarrier per slot), R - 3 macro rows ahead.  Each union value is one LDS of NQ
// doubles from the staged window; the coefficients are constant-bank operands,
// each feeding NQ FMAs.
// One macro-row step of k_residual_mac for the rows [T0, T1) of the half-warp's macro
// (PART: compile-time row set, so only its accumulators are live).
template <int K, int NQ, int MX, int R, int PART>
__device__ __forceinline__ void mac_step(const MacArgs &P, double *ring, uint64_t *full, double *prevq, int Lx,
                                         int Ly, int64_t NT, int JS, const uint8_t *__restrict__ rcls,
                                         const double *__restrict__ b, double *__restrict__ r, int apply, int c,
                                         int jj, int jm, int lo, int im, int mloc, int sl, int N, bool active) {
  using W = VT<NQ>;
  using V = typename W::T;
  constexpr int SPC = 16;
  constexpr int VPC = SPC * NQ;
  constexpr int RWX = K * MX + 2 * K;
  constexpr int GROUP = K * RWX * VPC;
  constexpr int KK = K * K;
  // PART 0: rows of line b = 0; 1: lines b >= 1; 2: every row of the macro
  constexpr int T0 = (K == 1 || PART != 1) ? 0 : K, T1 = (K == 1 || PART != 0) ? KK : K;
  const int n = c * SPC + sl;
  const bool valid = n < N;
  const int64_t tg = (int64_t)(valid ? n : N - 1) * NQ;
    // row classes (lane t of each half: row t) and b, issued before the wait
    int rc = 0x100;
    if (active && sl < KK) {
      const int X = K * im + sl % K, Y = K * jm + sl / K;
      if (X < Lx && Y < Ly) rc = __ldg(rcls + (int64_t)Y * Lx + X);
    }
    V bv[KK];
#pragma unroll
    for (int t = 0; t < KK; ++t) {
      const int X = K * im + t % K, Y = K * jm + t / K;
      bv[t] = (t >= T0 && t < T1 && active && !apply && X < Lx && Y < Ly)
                  ? W::ld(b + ((int64_t)Y * Lx + X) * NT + tg)
                  : W::zero();
    }
#pragma unroll
    for (int g = 0; g < 3; ++g) mbar_wait(&full[(lo + g) % R], (unsigned)(((lo + g) / R) & 1));
    {
      const double *gp[3];
#pragma unroll
      for (int g = 0; g < 3; ++g) gp[g] = ring + (size_t)((lo + g) % R) * GROUP + (K * mloc) * VPC + sl * NQ;
      auto ld = [&](int yl, int xl) -> V {  // window line yl = dy + K, column xl = dx + K
        const double *p = gp[yl / K] + ((yl % K) * RWX + xl) * VPC;
        if constexpr (NQ == 2) return *reinterpret_cast<const double2 *>(p);
        else if constexpr (NQ == 1) return *p;
        else if constexpr (NQ == 3) return V3{p[0], p[1], p[2]};  // shared memory: plain loads, not __ldg
        else return V4{*reinterpret_cast<const double2 *>(p), *reinterpret_cast<const double2 *>(p + 2)};
      };
      V am[KK], ak[KK];
#pragma unroll
      for (int t = 0; t < KK; ++t) am[t] = ak[t] = W::zero();
      mac_accum_ld_part<K>(PART, ld, P.C, am, ak);
      const double *pqr = prevq + (((size_t)(c & 1) * MX + mloc) * JS + jj) * KK;
      double *pqw = prevq + (((size_t)((c + 1) & 1) * MX + mloc) * JS + jj) * KK;
#pragma unroll
      for (int t = 0; t < KK; ++t) {
        if (t < T0 || t >= T1) continue;  // compile time: the other part's rows
        const int cls = __shfl_sync(0xffffffffu, rc, t, 16);
        const double lastq = W::get(am[t], NQ - 1);
        double jmv = __shfl_up_sync(0xffffffffu, lastq, 1, 16);
        if (sl == 0) jmv = pqr[t];
        if (sl == SPC - 1) pqw[t] = lastq;
        double o[NQ];
#pragma unroll
        for (int a = 0; a < NQ; ++a) {
          double acc = W::get(bv[t], a);
#pragma unroll
          for (int c2 = 0; c2 < NQ; ++c2)
            acc -= P.CE[a * NQ + c2] * W::get(am[t], c2) + P.Mt[a * NQ + c2] * W::get(ak[t], c2);
          if (a == 0 && n > 0) acc += jmv;
          o[a] = apply ? -acc : acc;
        }
        if (cls == 0xFF) {  // constrained row: identity
          const V own = ld(t / K + K, t % K + K);
#pragma unroll
          for (int a = 0; a < NQ; ++a) o[a] = apply ? W::get(own, a) : W::get(bv[t], a) - W::get(own, a);
        }
        const int X = K * im + t % K, Y = K * jm + t / K;
        if (active && valid && cls <= 0xFF) W::st(r + ((int64_t)Y * Lx + X) * NT + tg, o);
      }
    }
}

template <int K, int NQ, int MX, int R, bool SPLIT = true>
__global__ void __launch_bounds__(16 * MX * (K > 1 && SPLIT ? 2 : 1)) k_residual_mac(const __grid_constant__ CUtensorMap umap,
                                                          const __grid_constant__ MacArgs P, int Lx, int Ly,
                                                          int64_t NT, int nstrips, int nmy, int JS,
                                                          const uint8_t *__restrict__ rcls,
                                                          const double *__restrict__ b, double *__restrict__ r,
                                                          int apply) {
  using W = VT<NQ>;
  using V = typename W::T;
  constexpr int SPC = 16;              // slabs per chunk
  constexpr int VPC = SPC * NQ;        // values per node and chunk
  constexpr int RWX = K * MX + 2 * K;  // staged window width (nodes)
  constexpr int GROUP = K * RWX * VPC; // doubles per group of K node lines
  constexpr int KK = K * K;
  constexpr int LA = R - 3;            // macro rows of TMA lookahead
  extern __shared__ __align__(128) double ring[];
  __shared__ __align__(8) uint64_t full[R];
  double *prevq = ring + R * GROUP;  // [2][MX][JS][KK]: (M u)_{last slab}[q] of the previous chunk (by parity)
  constexpr int NPART = K > 1 && SPLIT ? 2 : 1;  // warps per macro pair: rows of line b = 0 / lines b >= 1
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int part = w % NPART, pw = w / NPART;
  const int h = lane >> 4, sl = lane & 15;
  const int strip = blockIdx.x % nstrips, seg = blockIdx.x / nstrips;
  const int j0 = seg * JS, ns = min(nmy, j0 + JS) - j0;  // macro rows of this segment
  const int x0 = K * MX * strip;                           // first node column of the strip
  const int mloc = 2 * pw + h;                             // this half-warp's macro within the strip
  const int im = MX * strip + mloc;
  const int ngrp = ns + 2;                                 // line groups per chunk (halo groups included)
  const int N = (int)(NT / NQ);
  const int nch = (N + SPC - 1) / SPC;
  const int nsteps = nch * ns;
  if (ns <= 0) return;
  if (tid == 0) {
    for (int z = 0; z < R; ++z) mbar_init(&full[z], 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  for (int e = tid; e < 2 * MX * JS * KK; e += blockDim.x) prevq[e] = 0.0;
  __syncthreads();
  constexpr unsigned kBytes = (unsigned)(GROUP * sizeof(double));
  auto issue = [&](int F) {
    const int c = F / ngrp, g = F - c * ngrp, z = F % R;
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    mbar_expect_tx(&full[z], kBytes);
    tma_load_3d(ring + (size_t)z * GROUP, &umap, c * VPC, x0 - K, K * (j0 + g - 1), &full[z]);
  };
  int issued = 0;  // groups issued so far (thread 0's bookkeeping)
  const bool active = im * K < Lx;
  for (int s = 0; s < nsteps; ++s) {
    const int c = s / ns, jj = s - c * ns, jm = j0 + jj;
    const int lo = c * ngrp + jj;  // first of the three groups of this step
    if (tid == 0) {  // keep the ring up to LA macro rows ahead, as far as free slots allow
      const int st = min(nsteps - 1, s + LA);
      const int hi = (st / ns) * ngrp + (st - (st / ns) * ns) + 2;
      while (issued <= hi && issued - R < lo) issue(issued++);
    }
    if (NPART == 1 && K > 1)
      mac_step<K, NQ, MX, R, 2>(P, ring, full, prevq, Lx, Ly, NT, JS, rcls, b, r, apply, c, jj, jm, lo, im, mloc, sl, N,
                                active);
    else if (part == 0)
      mac_step<K, NQ, MX, R, 0>(P, ring, full, prevq, Lx, Ly, NT, JS, rcls, b, r, apply, c, jj, jm, lo, im, mloc, sl, N,
                                active);
    else
      mac_step<K, NQ, MX, R, 1>(P, ring, full, prevq, Lx, Ly, NT, JS, rcls, b, r, apply, c, jj, jm, lo, im, mloc, sl, N,
                                active);
    __syncthreads();  // every warp is done with this step's groups before their slots are refilled
  }
}

template <int K, int NQ, int MX, int R, bool SPLIT = true>
bool mac_launch(const Level &L, int N, const MacArgs &P, const double *u, const double *b, double *r, int apply,
                cudaStream_t s) {
  constexpr int VPC = 16 * NQ;
  constexpr int RWX = K * MX + 2 * K;
  const int64_t NT = (int64_t)N * NQ;
  CUtensorMap umap;
  if (!umap_for(u, NT, L.Lx, L.Ly, VPC, RWX, &umap, K)) return false;
  const int nmx = (L.Lx + K - 1) / K, nmy = (L.Ly + K - 1) / K;
  const int nstrips = (nmx + MX - 1) / MX;
  // segments: enough CTAs for ~2 per SM, each walking all time chunks of its segment
  const int target = 2 * num_sms();
  int nseg = std::max(1, std::min(nmy, (target + nstrips - 1) / nstrips));
  const int JS = (nmy + nseg - 1) / nseg;
  nseg = (nmy + JS - 1) / JS;
  const size_t smem = ((size_t)R * K * RWX * VPC + (size_t)2 * MX * JS * K * K) * sizeof(double);
  if (smem > 200 * 1024) return false;
  smem_optin((const void *)k_residual_mac<K, NQ, MX, R, SPLIT>, (int)smem);
  k_residual_mac<K, NQ, MX, R, SPLIT><<<nstrips * nseg, 16 * MX * (K > 1 && SPLIT ? 2 : 1), smem, s>>>(umap, P, L.Lx, L.Ly, NT, nstrips, nmy, JS,
                                                                        L.rcls, b, r, apply);
  ++g_launches;
  return true;
}

template <int NQ>
void rows_launch(const Level &L, int N, const MacArgs &P, const double *u, const double *b, double *r, int apply,
                 cudaStream_t s) {
  const int nchunk = (N + 31) / 32;
  const int64_t warps = L.ngen_rows * nchunk;
  k_residual_rows<NQ><<<(unsigned)((warps + 7) / 8), 256, 0, s>>>(L.ngen_rows, L.gen_rows, N, L.rcls, u, b, r, P,
                                                                   L.stencil, L.goff, apply);
  ++g_launches;
}

}  // namespace

bool launch_residual_mac(const Level &L, int k, int q, int N, const Temporal &tm, const double *u, const double *b,
                         double *r, cudaStream_t s) {
  static const int mode = [] {  // WRMG_RESIDUAL=tile: the previous class-stencil kernels (A/B)
    const char *e = getenv("WRMG_RESIDUAL");
    return (e && std::string(e) == "tile") ? 0 : 1;
  }();
  if (!mode || !L.mac_ok || !L.stencil_ok || q > 3) return false;
  const int apply = b == nullptr;
  MacArgs P{};
  P.C = L.mac.C;
  for (int e = 0; e < tm.nq * tm.nq; ++e) {
    P.CE[e] = tm.CE[e];
    P.Mt[e] = tm.Mt[e];
  }
  bool ok = false;
  static const bool l1 = [] {  // WRMG_RESIDUAL=macl1: the L1 macro kernel (A/B)
    const char *e = getenv("WRMG_RESIDUAL");
    return e && std::string(e) == "macl1";
  }();
  if (!l1) {
#define WRMG_MAC(KK_, NQ_, MX_, R_) \
  if (k == KK_ && q + 1 == NQ_) ok = mac_launch<KK_, NQ_, MX_, R_>(L, N, P, u, b, r, apply, s);
    WRMG_MAC(1, 1, 16, 8) WRMG_MAC(1, 2, 16, 8) WRMG_MAC(1, 3, 16, 8) WRMG_MAC(1, 4, 16, 8)
    static const int k2mx = [] {  // P2 levels: 16 macro columns per CTA (C5 L7 residual 2.5 vs 2.1 TB/s
      const char *e = getenv("WRMG_MAC_K2");  // with 8); WRMG_MAC_K2=8 for the narrower form (A/B)
      return e ? atoi(e) : 16;
    }();
    static const bool k2split = [] {  // WRMG_MAC_K2_SPLIT=0: P2 macros without the two-warp row split (A/B)
      const char *e = getenv("WRMG_MAC_K2_SPLIT");
      return !(e && e[0] == '0');
    }();
    if (k == 2 && q == 1 && k2mx == 16 && !k2split) ok = mac_launch<2, 2, 16, 4, false>(L, N, P, u, b, r, apply, s);
    if (!ok && k2mx == 16) {
      WRMG_MAC(2, 2, 16, 4)
    }
    if (!ok) {
      WRMG_MAC(2, 1, 8, 5) WRMG_MAC(2, 2, 8, 5) WRMG_MAC(2, 3, 8, 5) WRMG_MAC(2, 4, 8, 4)
    }
    WRMG_MAC(3, 1, 8, 4) WRMG_MAC(3, 2, 8, 4)
#undef WRMG_MAC
  }
  if (!ok) {
#define WRMG_MACL1(KK_, NQ_) \
  if (k == KK_ && q + 1 == NQ_) ok = mac_l1_launch<KK_, NQ_>(L, N, P, u, b, r, apply, s);
    WRMG_MACL1(1, 1) WRMG_MACL1(1, 2) WRMG_MACL1(1, 3) WRMG_MACL1(1, 4)
    WRMG_MACL1(2, 1) WRMG_MACL1(2, 2) WRMG_MACL1(2, 3) WRMG_MACL1(2, 4)
    WRMG_MACL1(3, 1) WRMG_MACL1(3, 2) WRMG_MACL1(3, 3)
#undef WRMG_MACL1
  }
  if (!ok) return false;
  if (L.ngen_rows > 0) {
    switch (q) {
      case 0: rows_launch<1>(L, N, P, u, b, r, apply, s); break;
      case 1: rows_launch<2>(L, N, P, u, b, r, apply, s); break;
      case 2: rows_launch<3>(L, N, P, u, b, r, apply, s); break;
      default: rows_launch<4>(L, N, P, u, b, r, apply, s); break;
    }
  }
  return true;
}

// Host: the interior class of every row type (a, b) and its coefficients in the
// generated entry order; rows of other (non-constrained) classes go to the fix-up list.
bool plan_residual_mac(Level &L, int k, const std::vector<int32_t> &cnt, const std::vector<int32_t> &dI,
                       const std::vector<int32_t> &dJ, const std::vector<double> &m, const std::vector<double> &kk,
                       std::vector<int32_t> &gen_rows) {
  gen_rows.clear();
  if (k < 1 || k > 3 || L.nx < 4 || L.ny < 4 || !L.stencil_ok) return false;
  const int ntyp = k * k;
  const int *kcnt = k == 1 ? kMacCnt1 : k == 2 ? kMacCnt2 : kMacCnt3;
  const int *kbase = k == 1 ? kMacBase1 : k == 2 ? kMacBase2 : kMacBase3;
  auto off = [&](int t, int e, int d) -> int {
    return k == 1 ? kMacOff1[t][e][d] : k == 2 ? kMacOff2[t][e][d] : kMacOff3[t][e][d];
  };
  std::memset(&L.mac, 0, sizeof(L.mac));
  for (int t = 0; t < ntyp; ++t) {
    const int a = t % k, bb = t / k;
    const int64_t X = (int64_t)k * (L.nx / 2) + a, Y = (int64_t)k * (L.ny / 2) + bb;
    const int cls = L.h_rcls[Y * L.Lx + X];
    if (cls >= L.stencil.ncls) return false;
    if (cnt[cls] != kcnt[t]) return false;
    L.mac.canon[t] = cls;
    for (int e = 0; e < kcnt[t]; ++e) {
      int f = -1;
      for (int e2 = 0; e2 < cnt[cls]; ++e2)
        if (dI[cls * kStencilMaxE + e2] == off(t, e, 0) && dJ[cls * kStencilMaxE + e2] == off(t, e, 1)) f = e2;
      if (f < 0) return false;
      L.mac.C.m[kbase[t] + e] = m[cls * kStencilMaxE + f];
      L.mac.C.k[kbase[t] + e] = kk[cls * kStencilMaxE + f];
    }
  }
  for (int64_t i = 0; i < L.nnode; ++i) {
    const int cls = L.h_rcls[i];
    if (cls == 0xFF) continue;  // constrained: identity row, handled in the macro kernel
    const int t = (int)((i / L.Lx) % k) * k + (int)((i % L.Lx) % k);
    if (cls != L.mac.canon[t]) gen_rows.push_back((int32_t)i);
  }
  return true;
}

}  // namespace wrmg
