// Kronecker-diagonalised waveform-relaxation patch solves (H7 + H8 for the
// heat operator, and the coarse solve H11).
//
// The heat patch block is a Kronecker sum (tensor-product
// space-time discretisation; eq. heatfem):
//     D_p = (C + E0) (x) M_p + Mt (x) K_p,      L_p = -E1 (x) M_p,  E1 = e_0 e_q^T (R2),
// with M_p, K_p symmetric and M_p positive definite.  With the generalised
// eigenpairs K_p V = M_p V Lambda, V^T M_p V = I (computed once per patch
// translation class, k_kron_setup), the patch space-time system decouples into
// m_p independent temporal problems, one per spatial mode i:
//     (C + E0 + lambda_i Mt) w_{n,i} = ghat_{n,i} + e_0 y_{n-1,i},
//     ghat_n = (I (x) V^T) g_n,    x_n = (I (x) V) w_n,    y_{n,i} = w_{n,i}[q],
// because V^T M_p V = I turns the jump carry M_p x_{n-1}[q] into y_{n-1}.  With
// S_i = (C + E0 + lambda_i Mt)^{-1} and sigma_i = S_i[q][0], the end trace obeys
// the scalar affine recurrence  y_{n,i} = (S_i ghat_{n,i})[q] + sigma_i y_{n-1,i},
// solved for 32 slabs at once by a warp shuffle scan (lanes = slabs) and across
// 32-slab chunks through shared memory (warps = chunks).  This is an exact
// solve of A_p x = g (R9), the same operator the LU path factors; it differs
// from the LU result only by rounding.  Per (patch, slab) it costs
// 2 (q+1) m_p^2 + O((q+1)^2 m_p) FMAs instead of the LU solve's (q+1)^2 m_p^2 + m_p^2.
#include <cfloat>

#include <cstdlib>

#include "internal.h"

namespace wrmg {
namespace {

struct TMk {
  double CE[16], Mt[16];
};

__device__ __forceinline__ int csr_find_k(const int32_t *rowptr, const int32_t *col, int64_t i, int32_t j) {
  int lo = rowptr[i], hi = rowptr[i + 1] - 1;
  while (lo <= hi) {
    int mid = (lo + hi) >> 1;
    int32_t c = col[mid];
    if (c == j) return mid;
    if (c < j) lo = mid + 1;
    else hi = mid - 1;
  }
  return -1;
}

// One warp per class: generalised symmetric eigenproblem K v = lambda M v by
// Cholesky M = L L^T, C = L^-1 K L^-T, cyclic Jacobi C = Q Lambda Q^T, V = L^-T Q;
// then the per-mode temporal inverses S_i and multipliers sigma_i.
// Outputs (stride mp, pad modes zero): V[t][j][i] (row j = patch node),
// VT[t][i][j], S[t][i][nq*nq], sig[t][i].
template <int NT>
__global__ void __launch_bounds__(NT) k_kron_setup(const int32_t *__restrict__ rowptr, const int32_t *__restrict__ col,
                             const double *__restrict__ Mv, const double *__restrict__ Kv,
                             const int32_t *__restrict__ nodes_all, const int32_t *__restrict__ rep, int mp, int nq,
                             TMk tm, double *__restrict__ scratch, int ld, double *__restrict__ Vout,
                             double *__restrict__ VTout, double *__restrict__ Sout, double *__restrict__ sigout,
                             int32_t *__restrict__ info) {
  // NT threads per class: one warp for the patch classes, a whole CTA for the
  // (single, large) coarsest level
#define KSYNC() \
  do {                              \
    if (NT == 32) __syncwarp();     \
    else __syncthreads();           \
  } while (0)
  __shared__ double red_off[NT / 32], red_dia[NT / 32];
  const int t = blockIdx.x, lane = threadIdx.x;
  const int32_t *nodes = nodes_all + (rep ? (int64_t)rep[t] * mp : 0);
  int m = 0;
  while (m < mp && nodes[m] >= 0) ++m;
  double *A = scratch + (size_t)t * 3 * mp * mp;  // M -> L
  double *B = A + (size_t)mp * mp;                // K -> X -> C
  double *Q = B + (size_t)mp * mp;
  for (int e = lane; e < m * m; e += NT) {
    int i = e / m, j = e % m;
    int pos = csr_find_k(rowptr, col, nodes[i], nodes[j]);
    A[e] = pos >= 0 ? Mv[pos] : 0.0;
    B[e] = pos >= 0 ? Kv[pos] : 0.0;
    Q[e] = (i == j) ? 1.0 : 0.0;
  }
  KSYNC();
  int bad = 0;
  // Cholesky (lower, in place, row-major A[i*m+j], j <= i)
  for (int j = 0; j < m; ++j) {
    double d = A[j * m + j];
    for (int p = 0; p < j; ++p) d -= A[j * m + p] * A[j * m + p];
    if (!(d > 0.0)) bad = 1;
    d = sqrt(fmax(d, 1e-300));
    KSYNC();
    for (int i = j + 1 + lane; i < m; i += NT) {
      double s = A[i * m + j];
      for (int p = 0; p < j; ++p) s -= A[i * m + p] * A[j * m + p];
      A[i * m + j] = s / d;
    }
    KSYNC();
    if (lane == 0) A[j * m + j] = d;
    KSYNC();
  }
  // X = L^-1 K (columns in parallel), then C = L^-1 X^T
  for (int c = lane; c < m; c += NT)
    for (int i = 0; i < m; ++i) {
      double s = B[i * m + c];
      for (int p = 0; p < i; ++p) s -= A[i * m + p] * B[p * m + c];
      B[i * m + c] = s / A[i * m + i];
    }
  KSYNC();
  // transpose X in place, then apply L^-1 again (C = L^-1 X^T)
  for (int e = lane; e < m * m; e += NT) {
    int i = e / m, j = e % m;
    if (i < j) {
      double tmp = B[i * m + j];
      B[i * m + j] = B[j * m + i];
      B[j * m + i] = tmp;
    }
  }
  KSYNC();
  for (int c = lane; c < m; c += NT)
    for (int i = 0; i < m; ++i) {
      double s = B[i * m + c];
      for (int p = 0; p < i; ++p) s -= A[i * m + p] * B[p * m + c];
      B[i * m + c] = s / A[i * m + i];
    }
  KSYNC();
  for (int e = lane; e < m * m; e += NT) {  // symmetrise
    int i = e / m, j = e % m;
    if (i < j) {
      double s = 0.5 * (B[i * m + j] + B[j * m + i]);
      B[i * m + j] = s;
      B[j * m + i] = s;
    }
  }
  KSYNC();
  // cyclic Jacobi
  for (int sweep = 0; sweep < 60; ++sweep) {
    double off = 0.0, dia = 0.0;
    for (int e = lane; e < m * m; e += NT) {
      int i = e / m, j = e % m;
      if (i != j) off += B[e] * B[e];
      else dia += B[e] * B[e];
    }
    for (int o = 16; o; o >>= 1) {
      off += __shfl_xor_sync(0xffffffffu, off, o);
      dia += __shfl_xor_sync(0xffffffffu, dia, o);
    }
    if (NT > 32) {
      if ((lane & 31) == 0) {
        red_off[lane >> 5] = off;
        red_dia[lane >> 5] = dia;
      }
      __syncthreads();
      off = 0.0;
      dia = 0.0;
      for (int w = 0; w < NT / 32; ++w) {
        off += red_off[w];
        dia += red_dia[w];
      }
      __syncthreads();
    }
    if (off <= 1e-32 * dia) break;
    for (int p = 0; p < m - 1; ++p)
      for (int q = p + 1; q < m; ++q) {
        const double apq = B[p * m + q];
        if (fabs(apq) <= 1e-300) continue;
        const double app = B[p * m + p], aqq = B[q * m + q];
        const double theta = (aqq - app) / (2.0 * apq);
        const double tt = (theta >= 0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
        const double c = 1.0 / sqrt(tt * tt + 1.0), s = tt * c;
        KSYNC();
        for (int k2 = lane; k2 < m; k2 += NT) {  // columns p, q
          double akp = B[k2 * m + p], akq = B[k2 * m + q];
          B[k2 * m + p] = c * akp - s * akq;
          B[k2 * m + q] = s * akp + c * akq;
          double qkp = Q[k2 * m + p], qkq = Q[k2 * m + q];
          Q[k2 * m + p] = c * qkp - s * qkq;
          Q[k2 * m + q] = s * qkp + c * qkq;
        }
        KSYNC();
        for (int k2 = lane; k2 < m; k2 += NT) {  // rows p, q
          double apk = B[p * m + k2], aqk = B[q * m + k2];
          B[p * m + k2] = c * apk - s * aqk;
          B[q * m + k2] = s * apk + c * aqk;
        }
        KSYNC();
        if (lane == 0) {
          B[p * m + q] = 0.0;
          B[q * m + p] = 0.0;
        }
        KSYNC();
      }
  }
  // V = L^-T Q (columns in parallel): back substitution with L^T
  double *Vt = Vout + (size_t)t * mp * ld, *VTt = VTout + (size_t)t * mp * ld;
  for (int e = lane; e < mp * ld; e += NT) {
    Vt[e] = 0.0;
    VTt[e] = 0.0;
  }
  KSYNC();
  for (int c = lane; c < m; c += NT)
    for (int i = m - 1; i >= 0; --i) {
      double s = Q[i * m + c];
      for (int p = i + 1; p < m; ++p) s -= A[p * m + i] * Q[p * m + c];
      Q[i * m + c] = s / A[i * m + i];
    }
  KSYNC();
  for (int e = lane; e < m * m; e += NT) {
    int j = e / m, i = e % m;  // node j, mode i
    Vt[j * ld + i] = Q[e];
    VTt[i * ld + j] = Q[e];
  }
  // per mode: S_i = (CE + lambda_i Mt)^-1 by Gauss-Jordan with partial pivoting
  for (int i = lane; i < mp; i += NT) {
    const double lam = i < m ? B[i * m + i] : 0.0;
    double a[16], inv[16];
    for (int r = 0; r < nq; ++r)
      for (int c = 0; c < nq; ++c) {
        a[r * nq + c] = tm.CE[r * nq + c] + lam * tm.Mt[r * nq + c];
        inv[r * nq + c] = (r == c) ? 1.0 : 0.0;
      }
    for (int c = 0; c < nq; ++c) {
      int pr = c;
      for (int r = c + 1; r < nq; ++r)
        if (fabs(a[r * nq + c]) > fabs(a[pr * nq + c])) pr = r;
      for (int c2 = 0; c2 < nq; ++c2) {
        double x = a[c * nq + c2]; a[c * nq + c2] = a[pr * nq + c2]; a[pr * nq + c2] = x;
        x = inv[c * nq + c2]; inv[c * nq + c2] = inv[pr * nq + c2]; inv[pr * nq + c2] = x;
      }
      const double d = a[c * nq + c];
      if (d == 0.0) bad = 1;
      for (int c2 = 0; c2 < nq; ++c2) {
        a[c * nq + c2] /= d;
        inv[c * nq + c2] /= d;
      }
      for (int r = 0; r < nq; ++r)
        if (r != c) {
          const double f = a[r * nq + c];
          for (int c2 = 0; c2 < nq; ++c2) {
            a[r * nq + c2] -= f * a[c * nq + c2];
            inv[r * nq + c2] -= f * inv[c * nq + c2];
          }
        }
    }
    for (int e = 0; e < nq * nq; ++e) Sout[((size_t)t * mp + i) * nq * nq + e] = inv[e];
    sigout[(size_t)t * mp + i] = inv[(nq - 1) * nq + 0];
  }
  if (NT == 32)
    bad = __any_sync(0xffffffffu, bad);
  else
    bad = __syncthreads_or(bad);
  if (lane == 0) info[t] = bad;
#undef KSYNC
}

// ------------------------------------------------------------------- sweep
// CTA = PP patches of one class x C chunks of 32 slabs (warp w: patch w / C,
// chunk w % C).  Lanes are slabs: gathers and scatters touch 32 (q+1)
// contiguous doubles per patch node (waveform-major layout, R4).
template <int NQ, int MP>
__global__ void __launch_bounds__(256, 2) k_sweep_kron(int N, int C, int PP, const int32_t *__restrict__ cta_patch,
                                                    const int32_t *__restrict__ cta_type,
                                                    const int32_t *__restrict__ pnodes,
                                                    const double *__restrict__ Vg, const double *__restrict__ VTg,
                                                    const double *__restrict__ Sg, const double *__restrict__ sigg,
                                                    const double *__restrict__ wnode, double omega,
                                                    const double *__restrict__ r, double *__restrict__ u) {
  constexpr int MPS = (MP + 1) & ~1;  // even row stride: 16-byte aligned rows for LDS.128
  extern __shared__ double sm[];
  double *sV = sm;                  // MP*MPS  V[j][i]
  double *sVT = sV + MP * MPS;      // MP*MPS  V^T[i][j]
  double *sS = sVT + MP * MPS;      // MP*NQ*NQ
  double *ssig = sS + MP * NQ * NQ; // MP
  double *swt = ssig + MP;          // PP*MP
  double *scar = swt + PP * MP;     // PP*C*MP chunk-end values
  int *snode = reinterpret_cast<int *>(scar + PP * C * MP);  // PP*MP
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int cta = blockIdx.x, ty = cta_type[cta];
  for (int e = tid; e < MP * MPS; e += blockDim.x) {
    sV[e] = Vg[(size_t)ty * MP * MPS + e];
    sVT[e] = VTg[(size_t)ty * MP * MPS + e];
  }
  for (int e = tid; e < MP * NQ * NQ; e += blockDim.x) sS[e] = Sg[(size_t)ty * MP * NQ * NQ + e];
  for (int e = tid; e < MP; e += blockDim.x) ssig[e] = sigg[(size_t)ty * MP + e];
  // scan coefficients: sig_i^(2^k) and sig_i^(lane + 1), formed once per CTA by the
  // squarings / binary powering each warp formed per mode before (bit-identical)
  __shared__ double ssig2[5][MP];
  __shared__ double spw[MP * 32];
  for (int e = tid; e < MP * 32; e += blockDim.x) {
    const double sg = sigg[(size_t)ty * MP + (e >> 5)];
    const int ex = (e & 31) + 1;
    double pw = 1.0, bs = sg;
    for (int bit = 0; bit < 6; ++bit) {
      pw *= ((ex >> bit) & 1) ? bs : 1.0;
      bs *= bs;
    }
    spw[e] = pw;
    if ((e & 31) < 5) {
      double p = sg;
      for (int k = 0; k < (e & 31); ++k) p *= p;
      ssig2[e & 31][e >> 5] = p;
    }
  }
  for (int e = tid; e < PP * MP; e += blockDim.x) {
    const int pp = e / MP, j = e % MP;
    const int p = cta_patch[(size_t)cta * PP + pp];
    const int nd = p >= 0 ? pnodes[(size_t)p * MP + j] : -1;
    snode[e] = nd;
    swt[e] = nd >= 0 ? omega * wnode[nd] : 0.0;
  }
  __syncthreads();
  const int pp = w / C, c = w % C;
  const int *nodes = snode + pp * MP;
  const int64_t NT = (int64_t)N * NQ;
  const int n = c * 32 + lane;
  const bool valid = n < N;
  // 1. ghat = (I (x) V^T) g, one temporal node at a time
  double t[NQ][MP];
#pragma unroll
  for (int a = 0; a < NQ; ++a) {
    double g[MP];
#pragma unroll
    for (int j = 0; j < MP; ++j) {
      const int nd = nodes[j];
      g[j] = (nd >= 0 && valid) ? __ldg(r + (int64_t)nd * NT + (int64_t)n * NQ + a) : 0.0;
    }
#pragma unroll
    for (int i = 0; i < MP; ++i) t[a][i] = 0.0;
#pragma unroll
    for (int j = 0; j < MP; ++j) {
      const double2 *row = reinterpret_cast<const double2 *>(sV + j * MPS);
#pragma unroll
      for (int i2 = 0; i2 < MP / 2; ++i2) {
        const double2 v = row[i2];
        t[a][2 * i2] = fma(v.x, g[j], t[a][2 * i2]);
        t[a][2 * i2 + 1] = fma(v.y, g[j], t[a][2 * i2 + 1]);
      }
      if constexpr (MP % 2) t[a][MP - 1] = fma(sV[j * MPS + MP - 1], g[j], t[a][MP - 1]);
    }
  }
  // 2. per mode: t = S_i ghat, then the local scan of the end trace (carry-in 0)
#pragma unroll
  for (int i = 0; i < MP; ++i) {
    double gh[NQ];
#pragma unroll
    for (int a = 0; a < NQ; ++a) gh[a] = t[a][i];
#pragma unroll
    for (int a = 0; a < NQ; ++a) {
      double s = 0.0;
#pragma unroll
      for (int b2 = 0; b2 < NQ; ++b2) s = fma(sS[(i * NQ + a) * NQ + b2], gh[b2], s);
      t[a][i] = s;
    }
    double v = t[NQ - 1][i];
#pragma unroll
    for (int k = 0; k < 5; ++k) {
      const double o = __shfl_up_sync(0xffffffffu, v, 1 << k);
      if (lane >= (1 << k)) v = fma(ssig2[k][i], o, v);
    }
    t[NQ - 1][i] = v;
    if (lane == 31) scar[(pp * C + c) * MP + i] = v;
  }
  __syncthreads();
  // 3. carry across chunks, end traces, full mode solutions, back-transform, scatter
#pragma unroll
  for (int i = 0; i < MP; ++i) {
    const double sg = ssig[i];
    double s32 = sg;
#pragma unroll
    for (int d = 0; d < 5; ++d) s32 *= s32;
    double Y = 0.0;
    for (int c2 = 0; c2 < c; ++c2) Y = fma(s32, Y, scar[(pp * C + c2) * MP + i]);
    const double pw = spw[i * 32 + lane];
    const double y = fma(pw, Y, t[NQ - 1][i]);
    double yp = __shfl_up_sync(0xffffffffu, y, 1);
    if (lane == 0) yp = Y;
#pragma unroll
    for (int a = 0; a < NQ - 1; ++a) t[a][i] = fma(sS[(i * NQ + a) * NQ + 0], yp, t[a][i]);
    t[NQ - 1][i] = y;
  }
  double *ub = u + (int64_t)n * NQ;
#pragma unroll
  for (int a = 0; a < NQ; ++a) {
    double x[MP];
#pragma unroll
    for (int j = 0; j < MP; ++j) x[j] = 0.0;
#pragma unroll
    for (int i = 0; i < MP; ++i) {
      const double2 *row = reinterpret_cast<const double2 *>(sVT + i * MPS);
#pragma unroll
      for (int j2 = 0; j2 < MP / 2; ++j2) {
        const double2 v = row[j2];
        x[2 * j2] = fma(v.x, t[a][i], x[2 * j2]);
        x[2 * j2 + 1] = fma(v.y, t[a][i], x[2 * j2 + 1]);
      }
      if constexpr (MP % 2) x[MP - 1] = fma(sVT[i * MPS + MP - 1], t[a][i], x[MP - 1]);
    }
    if (valid) {
#pragma unroll
      for (int j = 0; j < MP; ++j) {
        const int nd = nodes[j];
        if (nd >= 0) atomicAdd(ub + (int64_t)nd * NT + a, swt[pp * MP + j] * x[j]);
      }
    }
  }
}


// ------------------------------------------------------------ sweep (DMMA)
// The two dense transforms of the Kronecker sweep, ghat = (I (x) V^T) g and
// x = (I (x) V) w, are small GEMMs per (patch, 16-slab chunk):
//     [modes x (slab, a)] = V^T [modes x nodes] * G [nodes x (slab, a)],
// issued on the FP64 tensor cores (mma.sync.m8n8k4.f64; tcgen05 has no FP64
// kind): one warp instruction = 256 FMAs instead of 32, which frees the issue
// slots the DFMA version spends on shared-memory operand traffic.  Fragment
// layout (verified by tools/dmma_layout.cu): a = A[l>>2][l&3], b = B[l&3][l>>2],
// c[e] = C[l>>2][2(l&3)+e].  In the C layout a lane holds one mode and one slab
// with both DG1 time values, so the per-mode 2x2 solve is lane-local and the end
// trace scan runs over the 4 lanes of a quad and the 4 column tiles.  DG1 only.
__device__ __forceinline__ void dmma(double &c0, double &c1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

__device__ __forceinline__ void cp_async16_zfill(void *smem, const void *gmem, bool valid) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  const int sz = valid ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa), "l"(gmem), "r"(sz) : "memory");
}

// Warp = one patch, walking its slabs in 16-slab chunks with the end-trace
// carry of every mode in registers (no inter-warp dependency, no barrier per
// patch); CTA = 8 patches of one translation class sharing the class factors in
// shared memory; persistent CTAs take patch groups in a strided order so the
// active window stays spatially compact (L2 reuse of shared patch nodes).  The
// gather of chunk c+1 (cp.async, zero-filled outside the lattice / horizon) is
// in flight while chunk c is transformed, solved and scattered.
template <int MP>
__global__ void __launch_bounds__(256, 2) k_sweep_kron_mma(int N, int ld, int ngroups,
                                                        const int32_t *__restrict__ grp_patch,
                                                        const int32_t *__restrict__ grp_type,
                                                        const int32_t *__restrict__ pnodes,
                                                        const double *__restrict__ Vg, const double *__restrict__ Sg,
                                                        const double *__restrict__ sigg,
                                                        const double *__restrict__ wnode, double omega,
                                                        const double *__restrict__ r, double *__restrict__ u) {
  constexpr int NQ = 2;
  constexpr int MT = (MP + 7) / 8;  // mode / node tiles of 8
  constexpr int KF = (MP + 3) / 4;  // k-steps of 4 over nodes (fwd) and modes (bwd)
  constexpr int P8 = 8 * MT;        // padded modes / nodes
  constexpr int K4 = 4 * KF;        // rows of the gathered tile (nodes) and of W (modes)
  // Padding chosen for conflict-free 64-bit fragment loads (a half-warp reads rows
  // q4 = 0..3 x columns g8 = 0..3): row strides = 4 or 12 (mod 16) doubles put the
  // four rows in disjoint bank groups.
  constexpr int LDV = P8 + 4;
  constexpr int LDG = 36;           // 32 (slab, a) columns + pad, 16-byte aligned rows
  constexpr int WPC = 8;            // warps (patches) per CTA
  extern __shared__ __align__(16) double sm[];
  double *sV = sm;                     // P8 x LDV: V[node][mode], zero padded
  double *sS = sV + P8 * LDV;          // P8 x 4: S_i (2x2)
  double *ssig = sS + P8 * 4;          // P8 x 4: sigma, sigma^2, sigma^4, (unused)
  double *sG = ssig + 4 * P8;          // WPC x 2 x K4 x LDG: gathered g, then W
  const int tid = threadIdx.x, l = tid & 31, w = tid >> 5;
  const int q4 = l & 3, g8 = l >> 2, qb = l & ~3;
  const int64_t NT = (int64_t)N * NQ;
  const int nch = (N + 15) / 16;
  double *Gw = sG + w * 2 * K4 * LDG;
  auto gather = [&](int p, int ch, double *G) {
    const int n0 = 16 * ch;
#pragma unroll
    for (int t = 0; t < K4 / 2; ++t) {  // K4 rows x 16 pieces of 16 bytes
      const int e = l + 32 * t, row = e >> 4, pc = e & 15;
      const int nd = row < MP ? __ldg(pnodes + (size_t)p * MP + row) : -1;
      const bool ok = nd >= 0 && n0 + pc < N;
      const double *src = ok ? r + (int64_t)nd * NT + (int64_t)(n0 + pc) * NQ : r;
      cp_async16_zfill(G + row * LDG + 2 * pc, src, ok);
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  };
  int cur_ty = -1;
  for (int grp = blockIdx.x; grp < ngroups; grp += gridDim.x) {
    const int ty = grp_type[grp];
    if (ty != cur_ty) {  // uniform across the CTA
      __syncthreads();
      for (int e = tid; e < P8 * P8; e += blockDim.x) {
        const int j = e / P8, i = e - j * P8;
        sV[j * LDV + i] = (j < MP && i < MP) ? Vg[((size_t)ty * MP + j) * ld + i] : 0.0;
      }
      for (int e = tid; e < P8 * 4; e += blockDim.x)
        sS[e] = (e >> 2) < MP ? Sg[((size_t)ty * MP + (e >> 2)) * 4 + (e & 3)] : 0.0;
      for (int i = tid; i < P8; i += blockDim.x) {
        const double sg = i < MP ? sigg[(size_t)ty * MP + i] : 0.0, sg2 = sg * sg;
        ssig[4 * i] = sg;
        ssig[4 * i + 1] = sg2;
        ssig[4 * i + 2] = sg2 * sg2;
        ssig[4 * i + 3] = 0.0;
      }
      cur_ty = ty;
      __syncthreads();
    }
    const int p = grp_patch[grp * WPC + w];
    if (p < 0) continue;
    // scatter targets of this lane: node 8mt + g8
    int snd[MT];
    double swj[MT];
#pragma unroll
    for (int mt = 0; mt < MT; ++mt) {
      const int j = 8 * mt + g8;
      snd[mt] = j < MP ? __ldg(pnodes + (size_t)p * MP + j) : -1;
      swj[mt] = snd[mt] >= 0 ? omega * __ldg(wnode + snd[mt]) : 0.0;
    }
    double Ycar[MT];
#pragma unroll
    for (int mt = 0; mt < MT; ++mt) Ycar[mt] = 0.0;
    gather(p, 0, Gw);
    for (int ch = 0; ch < nch; ++ch) {
      double *G = Gw + (ch & 1) * K4 * LDG;
      if (ch + 1 < nch) {
        gather(p, ch + 1, Gw + ((ch + 1) & 1) * K4 * LDG);
        asm volatile("cp.async.wait_group 1;\n" ::: "memory");
      } else {
        asm volatile("cp.async.wait_group 0;\n" ::: "memory");
      }
      __syncwarp();
      // 1. forward transform on the tensor cores: acc[mt][nt] = (V^T G)[8mt + g8][8nt + 2 q4 + e]
      double acc[MT][4][2];
#pragma unroll
      for (int mt = 0; mt < MT; ++mt)
#pragma unroll
        for (int nt = 0; nt < 4; ++nt) acc[mt][nt][0] = acc[mt][nt][1] = 0.0;
#pragma unroll
      for (int kk = 0; kk < KF; ++kk) {
        double bf[4];
#pragma unroll
        for (int nt = 0; nt < 4; ++nt) bf[nt] = G[(4 * kk + q4) * LDG + 8 * nt + g8];
#pragma unroll
        for (int mt = 0; mt < MT; ++mt) {
          const double a = sV[(4 * kk + q4) * LDV + 8 * mt + g8];
#pragma unroll
          for (int nt = 0; nt < 4; ++nt) dmma(acc[mt][nt][0], acc[mt][nt][1], a, bf[nt]);
        }
      }
      // 2. per mode: t = S_i ghat; end-trace scan over the quad's 4 slabs and the 4 column tiles,
      //    carried in from the previous chunk; w = (t0 + S_i[0][0] y_{n-1}, y_n)
#pragma unroll
      for (int mt = 0; mt < MT; ++mt) {
        const int i = 8 * mt + g8;
        const double s00 = sS[i * 4 + 0], s01 = sS[i * 4 + 1], s10 = sS[i * 4 + 2], s11 = sS[i * 4 + 3];
        const double sg = ssig[4 * i], sg2 = ssig[4 * i + 1], sg4 = ssig[4 * i + 2];
        const double pw = q4 == 0 ? sg : q4 == 1 ? sg2 : q4 == 2 ? sg2 * sg : sg4;  // sg^(q4+1)
        double Y = Ycar[mt];
#pragma unroll
        for (int nt = 0; nt < 4; ++nt) {
          const double g0 = acc[mt][nt][0], g1 = acc[mt][nt][1];
          const double t0 = fma(s00, g0, s01 * g1);
          double v = fma(s10, g0, s11 * g1);
          double o = __shfl_up_sync(0xffffffffu, v, 1);
          v = fma(q4 >= 1 ? sg : 0.0, o, v);
          o = __shfl_up_sync(0xffffffffu, v, 2);
          v = fma(q4 >= 2 ? sg2 : 0.0, o, v);
          const double y = fma(pw, Y, v);
          double yp = __shfl_up_sync(0xffffffffu, y, 1);
          if (q4 == 0) yp = Y;
          acc[mt][nt][0] = fma(s00, yp, t0);
          acc[mt][nt][1] = y;
          Y = __shfl_sync(0xffffffffu, y, qb | 3);
        }
        Ycar[mt] = Y;
      }
      // 3. W (modes < K4) -> this chunk's gather buffer, then the backward transform
      __syncwarp();
#pragma unroll
      for (int mt = 0; mt < MT; ++mt) {
        const int i = 8 * mt + g8;
        if (i < K4)
#pragma unroll
          for (int nt = 0; nt < 4; ++nt)
            *reinterpret_cast<double2 *>(G + i * LDG + 8 * nt + 2 * q4) =
                make_double2(acc[mt][nt][0], acc[mt][nt][1]);
      }
      __syncwarp();
#pragma unroll
      for (int mt = 0; mt < MT; ++mt)
#pragma unroll
        for (int nt = 0; nt < 4; ++nt) acc[mt][nt][0] = acc[mt][nt][1] = 0.0;
#pragma unroll
      for (int kk = 0; kk < KF; ++kk) {
        double bw[4];
#pragma unroll
        for (int nt = 0; nt < 4; ++nt) bw[nt] = G[(4 * kk + q4) * LDG + 8 * nt + g8];
#pragma unroll
        for (int mt = 0; mt < MT; ++mt) {
          const double a = sV[(8 * mt + g8) * LDV + 4 * kk + q4];
#pragma unroll
          for (int nt = 0; nt < 4; ++nt) dmma(acc[mt][nt][0], acc[mt][nt][1], a, bw[nt]);
        }
      }
      __syncwarp();  // W reads done before the buffer is refilled two chunks later
      // 4. weighted additive scatter: lane holds node 8mt + g8, slab 16ch + 4nt + q4, both a
#pragma unroll
      for (int mt = 0; mt < MT; ++mt) {
        const int nd = snd[mt];
        if (nd < 0) continue;
        const double wj = swj[mt];
#pragma unroll
        for (int nt = 0; nt < 4; ++nt) {
          const int n = 16 * ch + 4 * nt + q4;
          if (n < N) {
            double *dst = u + (int64_t)nd * NT + (int64_t)n * NQ;
            atomicAdd(dst, wj * acc[mt][nt][0]);
            atomicAdd(dst + 1, wj * acc[mt][nt][1]);
          }
        }
      }
    }
  }
}

template <int MP>
void sweep_kron_mma_launch(const Level &L, int N, const double *r, double *u, double omega, cudaStream_t s,
                           int ngroups, const int32_t *grp_patch, const int32_t *grp_type) {
  constexpr int P8 = 8 * ((MP + 7) / 8);
  constexpr int K4 = 4 * ((MP + 3) / 4);
  const size_t smem = (size_t)(P8 * (P8 + 4) + P8 * 4 + 4 * P8 + 8 * 2 * K4 * 36) * sizeof(double);
  smem_optin((const void *)k_sweep_kron_mma<MP>, 220 * 1024);
  const int grid = std::min(ngroups, num_sms() * 2);
  k_sweep_kron_mma<MP><<<grid, 256, smem, s>>>(N, (L.mp + 1) & ~1, ngroups, grp_patch, grp_type, L.pnodes,
                                               L.kV, L.kS, L.ksig, L.wnode, omega, r, u);
  ++g_launches;
}

template <int NQ, int MP>
void sweep_kron_launch(const Level &L, int N, const double *r, double *u, double omega, cudaStream_t s, int ncta,
                       int PP, const int32_t *cta_patch, const int32_t *cta_type) {
  const int C = (N + 31) / 32;
  constexpr int MPS = (MP + 1) & ~1;
  size_t smem = (size_t)(2 * MP * MPS + MP * NQ * NQ + MP + PP * MP + PP * C * MP) * sizeof(double) +
                (size_t)PP * MP * sizeof(int);
  smem_optin((const void *)k_sweep_kron<NQ, MP>, 200 * 1024);
  k_sweep_kron<NQ, MP><<<ncta, 32 * C * PP, smem, s>>>(N, C, PP, cta_patch, cta_type, L.pnodes, L.kV,
                                                               L.kVT, L.kS, L.ksig, L.wnode, omega, r, u);
  ++g_launches;
}

// ------------------------------------------------------------- coarse (kron)
// z-transform: T[n][a][i] = (S_i (V^T g_n)[:, i])[a] for every slab (block n).
__global__ void __launch_bounds__(256) k_ckron_fwd(int mp, int nq, int64_t NT, const int32_t *__restrict__ nodes,
                                                   const double *__restrict__ V, const double *__restrict__ S,
                                                   const double *__restrict__ r, double *__restrict__ T) {
  extern __shared__ double g[];  // nq * mp
  const int n = blockIdx.x;
  for (int e = threadIdx.x; e < nq * mp; e += blockDim.x) {
    const int a = e / mp, j = e % mp;
    g[e] = r[(int64_t)nodes[j] * NT + (int64_t)n * nq + a];
  }
  __syncthreads();
  for (int i = threadIdx.x; i < mp; i += blockDim.x) {
    double gh[4] = {0, 0, 0, 0};
    for (int j = 0; j < mp; ++j) {
      const double v = V[(int64_t)j * mp + i];
      for (int a = 0; a < nq; ++a) gh[a] = fma(v, g[a * mp + j], gh[a]);
    }
    for (int a = 0; a < nq; ++a) {
      double s = 0.0;
      for (int b = 0; b < nq; ++b) s = fma(S[((int64_t)i * nq + a) * nq + b], gh[b], s);
      T[((int64_t)n * nq + a) * mp + i] = s;
    }
  }
}

// Variants for mp <= 128 and compile-time NQ: thread (i = t % 128, half = t / 128)
// sums half of the j range with 4 independent loads in flight; halves combined in
// shared memory.  The generic kernels above keep one thread per mode and a serial
// j loop (latency-bound on the V loads: ~55 us per call at C2's 121 coarse modes).
template <int NQ>
__global__ void __launch_bounds__(256) k_ckron_fwd2(int mp, int64_t NT, const int32_t *__restrict__ nodes,
                                                    const double *__restrict__ V, const double *__restrict__ S,
                                                    const double *__restrict__ r, double *__restrict__ T) {
  extern __shared__ double g[];  // NQ * mp + 2 * NQ * 128
  double *ph = g + NQ * mp;
  const int n = blockIdx.x, tid = threadIdx.x, i = tid & 127, half = tid >> 7;
  for (int e = tid; e < NQ * mp; e += blockDim.x) {
    const int a = e / mp, j = e - a * mp;
    g[e] = r[(int64_t)nodes[j] * NT + (int64_t)n * NQ + a];
  }
  __syncthreads();
  double gh[NQ];
#pragma unroll
  for (int a = 0; a < NQ; ++a) gh[a] = 0.0;
  if (i < mp) {
    const int j0 = half * ((mp + 1) / 2), j1 = min(mp, j0 + (mp + 1) / 2);
    int j = j0;
    for (; j + 4 <= j1; j += 4) {
      double v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) v[u] = __ldg(V + (int64_t)(j + u) * mp + i);
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int a = 0; a < NQ; ++a) gh[a] = fma(v[u], g[a * mp + j + u], gh[a]);
    }
    for (; j < j1; ++j) {
      const double v = __ldg(V + (int64_t)j * mp + i);
#pragma unroll
      for (int a = 0; a < NQ; ++a) gh[a] = fma(v, g[a * mp + j], gh[a]);
    }
  }
#pragma unroll
  for (int a = 0; a < NQ; ++a) ph[(half * NQ + a) * 128 + i] = gh[a];
  __syncthreads();
  if (half == 0 && i < mp) {
#pragma unroll
    for (int a = 0; a < NQ; ++a) gh[a] = ph[a * 128 + i] + ph[(NQ + a) * 128 + i];
#pragma unroll
    for (int a = 0; a < NQ; ++a) {
      double sum = 0.0;
#pragma unroll
      for (int b = 0; b < NQ; ++b) sum = fma(S[((int64_t)i * NQ + a) * NQ + b], gh[b], sum);
      T[((int64_t)n * NQ + a) * mp + i] = sum;
    }
  }
}

template <int NQ>
__global__ void __launch_bounds__(256) k_ckron_bwd2(int mp, int64_t NT, const int32_t *__restrict__ nodes,
                                                    const double *__restrict__ VT, const double *__restrict__ T,
                                                    double *__restrict__ x) {
  extern __shared__ double w[];  // NQ * mp + 2 * NQ * 128
  double *ph = w + NQ * mp;
  const int n = blockIdx.x, tid = threadIdx.x, j = tid & 127, half = tid >> 7;
  for (int e = tid; e < NQ * mp; e += blockDim.x) w[e] = T[(int64_t)n * NQ * mp + e];
  __syncthreads();
  double xs[NQ];
#pragma unroll
  for (int a = 0; a < NQ; ++a) xs[a] = 0.0;
  if (j < mp) {
    const int i0 = half * ((mp + 1) / 2), i1 = min(mp, i0 + (mp + 1) / 2);
    int i = i0;
    for (; i + 4 <= i1; i += 4) {
      double v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) v[u] = __ldg(VT + (int64_t)(i + u) * mp + j);
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int a = 0; a < NQ; ++a) xs[a] = fma(v[u], w[a * mp + i + u], xs[a]);
    }
    for (; i < i1; ++i) {
      const double v = __ldg(VT + (int64_t)i * mp + j);
#pragma unroll
      for (int a = 0; a < NQ; ++a) xs[a] = fma(v, w[a * mp + i], xs[a]);
    }
  }
#pragma unroll
  for (int a = 0; a < NQ; ++a) ph[(half * NQ + a) * 128 + j] = xs[a];
  __syncthreads();
  if (half == 0 && j < mp)
#pragma unroll
    for (int a = 0; a < NQ; ++a)
      x[(int64_t)nodes[j] * NT + (int64_t)n * NQ + a] = ph[a * 128 + j] + ph[(NQ + a) * 128 + j];
}

// per-mode recurrence over all slabs: one warp per mode, lanes = slabs of a
// 32-slab chunk (shuffle scan), chunks in order with the end trace carried.
__global__ void k_ckron_scan(int N, int mp, int nq, const double *__restrict__ S, const double *__restrict__ sig,
                             double *__restrict__ T) {
  const int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (i >= mp) return;
  const double sg = sig[i];
  double pw = 1.0, bs = sg;
#pragma unroll
  for (int bit = 0; bit < 6; ++bit) {
    pw *= (((lane + 1) >> bit) & 1) ? bs : 1.0;
    bs *= bs;
  }
  double carry = 0.0;
  for (int n0 = 0; n0 < N; n0 += 32) {
    const int n = n0 + lane;
    const bool valid = n < N;
    double *Tn = T + (int64_t)n * nq * mp;
    double v = valid ? Tn[(nq - 1) * mp + i] : 0.0, p = sg;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const double o = __shfl_up_sync(0xffffffffu, v, d);
      v = fma(lane >= d ? p : 0.0, o, v);
      p *= p;
    }
    const double y = fma(pw, carry, v);
    double yp = __shfl_up_sync(0xffffffffu, y, 1);
    if (lane == 0) yp = carry;
    if (valid) {
      for (int a = 0; a < nq - 1; ++a) Tn[a * mp + i] = fma(S[((int64_t)i * nq + a) * nq + 0], yp, Tn[a * mp + i]);
      Tn[(nq - 1) * mp + i] = y;
    }
    carry = __shfl_sync(0xffffffffu, y, 31);
  }
}

__global__ void __launch_bounds__(256) k_ckron_bwd(int mp, int nq, int64_t NT, const int32_t *__restrict__ nodes,
                                                   const double *__restrict__ VT, const double *__restrict__ T,
                                                   double *__restrict__ x) {
  extern __shared__ double w[];  // nq * mp
  const int n = blockIdx.x;
  for (int e = threadIdx.x; e < nq * mp; e += blockDim.x) w[e] = T[(int64_t)n * nq * mp + e];
  __syncthreads();
  for (int j = threadIdx.x; j < mp; j += blockDim.x) {
    double xs[4] = {0, 0, 0, 0};
    for (int i = 0; i < mp; ++i) {
      const double v = VT[(int64_t)i * mp + j];
      for (int a = 0; a < nq; ++a) xs[a] = fma(v, w[a * mp + i], xs[a]);
    }
    for (int a = 0; a < nq; ++a) x[(int64_t)nodes[j] * NT + (int64_t)n * nq + a] = xs[a];
  }
}

TMk make_tmk(const Temporal &T) {
  TMk t{};
  for (int e = 0; e < T.nq * T.nq; ++e) {
    t.CE[e] = T.CE[e];
    t.Mt[e] = T.Mt[e];
  }
  return t;
}

}  // namespace

void launch_kron_setup(const Level &L, int nq, const Temporal &tm, double *scratch, cudaStream_t s) {
  k_kron_setup<32><<<L.ntypes, 32, 0, s>>>(L.A.rowptr, L.A.col, L.A.val, L.A.val2, L.pnodes, L.type_rep, L.mp, nq,
                                       make_tmk(tm), scratch, (L.mp + 1) & ~1, L.kV, L.kVT, L.kS, L.ksig, L.info);
  ++g_launches;
}

void launch_kron_setup_coarse(const Level &L, Coarse &C, int nq, const Temporal &tm, double *scratch,
                              cudaStream_t s) {
  k_kron_setup<1024><<<1, 1024, 0, s>>>(L.A.rowptr, L.A.col, L.A.val, L.A.val2, C.nodes, nullptr, C.mp, nq,
                                         make_tmk(tm),
                                scratch, C.mp, C.kV, C.kVT, C.kS, C.ksig, C.info);
  ++g_launches;
}

bool launch_sweep_kron(const Level &L, int q, int N, const double *r, double *u, double omega, cudaStream_t s,
                       const SweepLists *sl) {
  const int nq = q + 1;
  const int ngrp8 = sl ? sl->ngrp8 : L.kron_ngrp8, ncta = sl ? sl->ncta : L.kron_ncta;
  const int pp = sl ? sl->pp : L.kron_pp;
  const int32_t *gp = sl ? sl->grp_patch8 : L.grp_patch8, *gt = sl ? sl->grp_type8 : L.grp_type8;
  const int32_t *cp = sl ? sl->cta_patch : L.cta_patch, *ct = sl ? sl->cta_type : L.cta_type;
  // Levels whose interior class runs in kernels_sweep_sym.cu leave only the boundary
  // classes here (a few hundred patches): the chunk-parallel kernel below (one warp per
  // 32-slab chunk) instead of the DMMA kernel's one warp walking all slabs of a patch
  // (latency-bound on so few patches).  WRMG_BOUNDARY_CP=0: the DMMA kernel (A/B).
  static const bool boundary_cp = [] {
    const char *e = getenv("WRMG_BOUNDARY_CP");
    return !(e && e[0] == '0');
  }();
  const bool residue = L.sym_ok && L.nsym > 0 && !sl && boundary_cp && N > 32;
  if (nq == 2 && L.npatch >= 1000 && !residue) {  // small levels: chunk-parallel kernel below
    if (L.mp == 19 || L.mp == 7 || L.mp == 1) {
      if (ngrp8 == 0) return true;  // nothing in this list
      if (L.mp == 19) sweep_kron_mma_launch<19>(L, N, r, u, omega, s, ngrp8, gp, gt);
      if (L.mp == 7) sweep_kron_mma_launch<7>(L, N, r, u, omega, s, ngrp8, gp, gt);
      if (L.mp == 1) sweep_kron_mma_launch<1>(L, N, r, u, omega, s, ngrp8, gp, gt);
      return true;
    }
  }
#define WRMG_SK(NQ, MP)                                                    \
  if (nq == NQ && L.mp == MP) {                                            \
    if (ncta > 0) sweep_kron_launch<NQ, MP>(L, N, r, u, omega, s, ncta, pp, cp, ct); \
    return true;                                                           \
  }
  WRMG_SK(1, 1) WRMG_SK(2, 1) WRMG_SK(3, 1) WRMG_SK(4, 1)
  WRMG_SK(1, 7) WRMG_SK(2, 7) WRMG_SK(3, 7) WRMG_SK(4, 7)
  WRMG_SK(1, 19) WRMG_SK(2, 19) WRMG_SK(3, 19)
#undef WRMG_SK
  return false;
}

void launch_coarse_solve_kron(const Coarse &C, const Level &L, int q, int N, const double *r, double *x,
                              cudaStream_t s) {
  const int nq = q + 1;
  const int64_t NT = (int64_t)N * nq;
  cudaMemsetAsync(x, 0, L.nnode * NT * sizeof(double), s);
  const size_t sm2 = (size_t)(nq * C.mp + 2 * nq * 128) * sizeof(double);
  const bool two = C.mp <= 128;
#define WRMG_CK(NQ, KER, ...)                                                 \
  case NQ: KER<NQ><<<N, 256, sm2, s>>>(__VA_ARGS__); break;
  if (two) {
    switch (nq) {
      WRMG_CK(1, k_ckron_fwd2, C.mp, NT, C.nodes, C.kV, C.kS, r, C.Z)
      WRMG_CK(2, k_ckron_fwd2, C.mp, NT, C.nodes, C.kV, C.kS, r, C.Z)
      WRMG_CK(3, k_ckron_fwd2, C.mp, NT, C.nodes, C.kV, C.kS, r, C.Z)
      default: k_ckron_fwd2<4><<<N, 256, sm2, s>>>(C.mp, NT, C.nodes, C.kV, C.kS, r, C.Z); break;
    }
  } else {
    k_ckron_fwd<<<N, 256, nq * C.mp * sizeof(double), s>>>(C.mp, nq, NT, C.nodes, C.kV, C.kS, r, C.Z);
  }
  ++g_launches;
  k_ckron_scan<<<(C.mp + 3) / 4, 128, 0, s>>>(N, C.mp, nq, C.kS, C.ksig, C.Z);
  ++g_launches;
  if (two) {
    switch (nq) {
      WRMG_CK(1, k_ckron_bwd2, C.mp, NT, C.nodes, C.kVT, C.Z, x)
      WRMG_CK(2, k_ckron_bwd2, C.mp, NT, C.nodes, C.kVT, C.Z, x)
      WRMG_CK(3, k_ckron_bwd2, C.mp, NT, C.nodes, C.kVT, C.Z, x)
      default: k_ckron_bwd2<4><<<N, 256, sm2, s>>>(C.mp, NT, C.nodes, C.kVT, C.Z, x); break;
    }
  } else {
    k_ckron_bwd<<<N, 256, nq * C.mp * sizeof(double), s>>>(C.mp, nq, NT, C.nodes, C.kVT, C.Z, x);
  }
#undef WRMG_CK
  ++g_launches;
}

}  // namespace wrmg
