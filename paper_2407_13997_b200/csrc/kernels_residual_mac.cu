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

template <int K, int NQ, int MX, int R>
__global__ void __launch_bounds__(32 * MX) k_residual_mac(const __grid_constant__ CUtensorMap umap,
                                                          const __grid_constant__ MacArgs P, int Lx, int Ly,
                                                          int64_t NT, int nstrips, int nmy, int JS,
                                                          const uint8_t *__restrict__ rcls,
                                                          const double *__restrict__ b, double *__restrict__ r,
                                                          int apply) {
  constexpr int VPC = NQ * (32 / NQ);  // time values per chunk (lanes >= VPC idle)
  constexpr int SPC = VPC / NQ;        // slabs per chunk
  constexpr int RWX = K * MX + 2 * K;  // staged window width (nodes)
  constexpr int GROUP = K * RWX * VPC; // doubles per group of K node lines
  constexpr int KK = K * K;
  constexpr int LA = R - 3;            // macro rows of TMA lookahead
  extern __shared__ __align__(128) double ring[];
  __shared__ __align__(8) uint64_t full[R];
  double *prevq = ring + R * GROUP;  // [2][MX][JS][KK]: (M u)_{last slab}[q] of the previous chunk (by parity)
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int strip = blockIdx.x % nstrips, seg = blockIdx.x / nstrips;
  const int j0 = seg * JS, ns = min(nmy, j0 + JS) - j0;  // macro rows of this segment
  const int x0 = K * MX * strip;                           // first node column of the strip
  const int im = MX * strip + w;                           // this warp's macro column
  const int ngrp = ns + 2;                                 // line groups per chunk (halo groups included)
  const int nch = (int)((NT + VPC - 1) / VPC);
  const int nsteps = nch * ns;
  if (ns <= 0) return;
  // lane constants: temporal node a of this lane; its column of (CE, Mt) (the lane's
  // contribution to every output a2 of its slab) or, for NQ = 3, its row
  const int al = lane % NQ, lbase = lane - al;
  double cea[NQ], mta[NQ];
#pragma unroll
  for (int c2 = 0; c2 < NQ; ++c2) {
    cea[c2] = (NQ & (NQ - 1)) ? P.CE[al * NQ + c2] : P.CE[c2 * NQ + al];
    mta[c2] = (NQ & (NQ - 1)) ? P.Mt[al * NQ + c2] : P.Mt[c2 * NQ + al];
  }
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
  // b and the row classes of a step, loaded one step ahead (software pipelined)
  auto load_b = [&](int st, double (&bvv)[KK], int &rcv) {
    const int cs = st / ns, jms = j0 + (st - cs * ns);
    const int64_t tgs = (int64_t)cs * VPC + lane;
    const bool vs = lane < VPC && tgs < NT;
    rcv = 0xFF;
    if (lane < KK) {
      const int X = K * im + lane % K, Y = K * jms + lane / K;
      rcv = (X < Lx && Y < Ly) ? (int)__ldg(rcls + (int64_t)Y * Lx + X) : 0x100;
    }
#pragma unroll
    for (int t = 0; t < KK; ++t) {
      const int X = K * im + t % K, Y = K * jms + t / K;
      bvv[t] = (vs && !apply && X < Lx && Y < Ly) ? __ldg(b + ((int64_t)Y * Lx + X) * NT + tgs) : 0.0;
    }
  };
  double bv[KK];
  int rc = 0xFF;
  if (active) load_b(0, bv, rc);
  for (int s = 0; s < nsteps; ++s) {
    const int c = s / ns, jj = s - c * ns, jm = j0 + jj;
    const int lo = c * ngrp + jj;  // first of the three groups of this step
    if (tid == 0) {  // keep the ring up to LA steps ahead, as far as free slots allow
      const int st = min(nsteps - 1, s + LA);
      const int hi = (st / ns) * ngrp + (st - (st / ns) * ns) + 2;
      while (issued <= hi && issued - R < lo) issue(issued++);
    }
    const int64_t tg = (int64_t)c * VPC + lane;
    const bool valid = lane < VPC && tg < NT;
    double bn[KK];
    int rcn = 0xFF;
    if (active && s + 1 < nsteps) load_b(s + 1, bn, rcn);
#pragma unroll
    for (int g = 0; g < 3; ++g) mbar_wait(&full[(lo + g) % R], (unsigned)(((lo + g) / R) & 1));
    if (active) {
      const double *gp[3];
#pragma unroll
      for (int g = 0; g < 3; ++g) gp[g] = ring + (size_t)((lo + g) % R) * GROUP + (K * w) * VPC + lane;
      double am[KK], ak[KK];
#pragma unroll
      for (int t = 0; t < KK; ++t) am[t] = ak[t] = 0.0;
      mac_accum<K, VPC, RWX>(gp[0], gp[1], gp[2], P.C, am, ak);
      const int n = c * SPC + lane / NQ;
      const double *pqr = prevq + (((size_t)(c & 1) * MX + w) * JS + jj) * KK;
      double *pqw = prevq + (((size_t)((c + 1) & 1) * MX + w) * JS + jj) * KK;
#pragma unroll
      for (int t = 0; t < KK; ++t) {
        const int cls = __shfl_sync(0xffffffffu, rc, t);
        if (cls > 0xFF) continue;  // outside the lattice
        const int X = K * im + t % K, Y = K * jm + t / K;
        // upwind jump (M u)_{n-1}[q]: lane - 1's value, lane 0 the previous chunk's last
        double jmv = __shfl_up_sync(0xffffffffu, am[t], 1);
        if (lane == 0) jmv = pqr[t];
        if (lane == VPC - 1) pqw[t] = am[t];
        double acc;
        if constexpr ((NQ & (NQ - 1)) == 0) {
          // reduce-scatter of the lanes' contributions over the NQ lanes of a slab
          double p[NQ];
#pragma unroll
          for (int a2 = 0; a2 < NQ; ++a2) p[a2] = fma(cea[a2], am[t], mta[a2] * ak[t]);
#pragma unroll
          for (int mm = NQ / 2; mm >= 1; mm >>= 1) {
#pragma unroll
            for (int j = 0; j < mm; ++j) {
              const bool hi = al & mm;
              const double send = hi ? p[j] : p[j + mm], keep = hi ? p[j + mm] : p[j];
              p[j] = keep + __shfl_xor_sync(0xffffffffu, send, mm);
            }
          }
          acc = bv[t] - p[0];
        } else {
          acc = bv[t];
#pragma unroll
          for (int c2 = 0; c2 < NQ; ++c2) {
            const double mc = __shfl_sync(0xffffffffu, am[t], (lbase + c2) & 31);
            const double kc = __shfl_sync(0xffffffffu, ak[t], (lbase + c2) & 31);
            acc -= cea[c2] * mc + mta[c2] * kc;
          }
        }
        if (al == 0 && n > 0) acc += jmv;
        double val = apply ? -acc : acc;  // apply: y = A u = -(0 - A u)
        if (cls == 0xFF) {
          const double own = gp[1][((t / K) * RWX + K + t % K) * VPC];
          val = apply ? own : bv[t] - own;
        }
        if (valid) r[((int64_t)Y * Lx + X) * NT + tg] = val;
      }
    }
    __syncthreads();  // every warp is done with this step's groups before their slots are refilled
#pragma unroll
    for (int t = 0; t < KK; ++t) bv[t] = bn[t];
    rc = rcn;
  }
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

template <int K, int NQ, int MX, int R>
bool mac_launch(const Level &L, int N, const MacArgs &P, const double *u, const double *b, double *r, int apply,
                cudaStream_t s) {
  constexpr int VPC = NQ * (32 / NQ);
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
  if (smem > 220 * 1024) return false;
  smem_optin((const void *)k_residual_mac<K, NQ, MX, R>, (int)smem);
  k_residual_mac<K, NQ, MX, R><<<nstrips * nseg, 32 * MX, smem, s>>>(umap, P, L.Lx, L.Ly, NT, nstrips, nmy, JS,
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
#define WRMG_MAC(KK_, NQ_, MX_, R_)                                   \
  if (k == KK_ && q + 1 == NQ_) ok = mac_launch<KK_, NQ_, MX_, R_>(L, N, P, u, b, r, apply, s);
  WRMG_MAC(1, 1, 8, 12) WRMG_MAC(1, 2, 8, 12) WRMG_MAC(1, 3, 8, 12) WRMG_MAC(1, 4, 8, 12)
  WRMG_MAC(2, 1, 8, 8) WRMG_MAC(2, 2, 8, 8) WRMG_MAC(2, 3, 8, 8) WRMG_MAC(2, 4, 8, 8)
  WRMG_MAC(3, 1, 4, 7) WRMG_MAC(3, 2, 4, 7) WRMG_MAC(3, 3, 4, 7) WRMG_MAC(3, 4, 4, 7)
#undef WRMG_MAC
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
