// Batched explicit inverses of large dense blocks (the coarse slab blocks of
// H11 once m reaches the hundreds: P2-P1 / P3-P2 on a 10x10 or 5x5 coarsest
// level, m_c up to 2048) by blocked Gauss-Jordan elimination with partial row
// pivoting (R10: first maximum |a|, singular when |pivot| < 1e-14 x the largest
// row sum of |a| of the input).
//
// Column-major m x m matrices.  Panels of NB columns [k0, k0 + nb):
//   K1 (k_gj_panel, one CTA per matrix): in-place Gauss-Jordan on the m x nb panel,
//      row swaps applied to the panel rows; the panel becomes
//      [P11^{-1} ; -A_O P11^{-1}] (pivot rows / other rows).
//   K2 (k_gj_swap_x): for every column outside the panel, the panel's row swaps,
//      X = its pivot rows, which are then zeroed.
//   K3 (k_gj_update, 64 x 64 tiles x matrices): A[:, j] += Panel X[:, j] for every
//      column outside the panel - the rank-nb update carrying 2 m^3 flops in all.
// After the last panel the columns are unscrambled in reverse pivot order
// (k_gj_unpermute, out of place).  The 1-column loop inside K1 is the only
// serial part; everything else is tile-parallel across all matrices.
#include "internal.h"
#include "ns_kernels.h"

namespace wrmg {
namespace {

constexpr int GJ_NB = 32;       // panel width
constexpr int GJ_T = 64;        // update tile (rows x columns)
constexpr int GJ_PTH = 1024;    // panel CTA

__global__ void __launch_bounds__(1024) k_gj_tol(const double *__restrict__ Aall, int m, double *__restrict__ tol,
                                                 int32_t *__restrict__ info) {
  __shared__ double sw[32];
  const double *A = Aall + (int64_t)blockIdx.x * m * m;
  double rn = 0.0;
  for (int r = threadIdx.x; r < m; r += blockDim.x) {
    double s = 0.0;
    for (int c = 0; c < m; ++c) s += fabs(A[(int64_t)c * m + r]);
    rn = fmax(rn, s);
  }
  for (int o = 16; o; o >>= 1) rn = fmax(rn, __shfl_xor_sync(0xffffffffu, rn, o));
  if ((threadIdx.x & 31) == 0) sw[threadIdx.x >> 5] = rn;
  __syncthreads();
  if (threadIdx.x == 0) {
    double mx = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) mx = fmax(mx, sw[w]);
    tol[blockIdx.x] = 1e-14 * mx;
    info[blockIdx.x] = 0;
  }
}

__global__ void __launch_bounds__(GJ_PTH) k_gj_panel(double *__restrict__ Aall, int m, int k0, int nb,
                                                      int32_t *__restrict__ pivall, int32_t *__restrict__ info,
                                                      const double *__restrict__ tol) {
  __shared__ double s_val[32];
  __shared__ int s_idx[32];
  __shared__ double s_row[GJ_NB];
  __shared__ double s_d;
  __shared__ int s_p;
  double *A = Aall + (int64_t)blockIdx.x * m * m;
  int32_t *piv = pivall + (int64_t)blockIdx.x * m;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, nw = blockDim.x >> 5;
  for (int t = 0; t < nb; ++t) {
    const int k = k0 + t;
    double bv = -1.0;
    int bi = m;
    for (int r = k + tid; r < m; r += blockDim.x) {
      const double v = fabs(A[(int64_t)k * m + r]);
      if (v > bv) {
        bv = v;
        bi = r;
      }
    }
    for (int o = 16; o; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ov > bv || (ov == bv && oi < bi)) {
        bv = ov;
        bi = oi;
      }
    }
    if (lane == 0) {
      s_val[wid] = bv;
      s_idx[wid] = bi;
    }
    __syncthreads();
    if (tid == 0) {
      double v = s_val[0];
      int ix = s_idx[0];
      for (int w = 1; w < nw; ++w)
        if (s_val[w] > v || (s_val[w] == v && s_idx[w] < ix)) {
          v = s_val[w];
          ix = s_idx[w];
        }
      s_p = ix;
      piv[k] = ix;
      if (v < tol[blockIdx.x] && info[blockIdx.x] == 0) info[blockIdx.x] = k + 1;
    }
    __syncthreads();
    const int p = s_p;
    if (tid < nb && p != k) {  // swap rows k, p in the panel columns
      double *cj = A + (int64_t)(k0 + tid) * m;
      const double tmp = cj[k];
      cj[k] = cj[p];
      cj[p] = tmp;
    }
    __syncthreads();
    if (tid == 0) s_d = A[(int64_t)k * m + k];
    __syncthreads();
    const double d = s_d;
    const double dinv = d != 0.0 ? 1.0 / d : 0.0;
    if (tid < nb) {  // scaled pivot row (panel columns)
      const double v = A[(int64_t)(k0 + tid) * m + k] * dinv;
      s_row[tid] = v;
    }
    __syncthreads();
    // other rows: A[i][j] -= A[i][k] * row_k[j]   (j != k in the panel)
    const int64_t tot = (int64_t)m * nb;
    for (int64_t e = tid; e < tot; e += blockDim.x) {
      const int i = (int)(e % m), jj = (int)(e / m);
      if (i == k || k0 + jj == k) continue;
      A[(int64_t)(k0 + jj) * m + i] -= A[(int64_t)k * m + i] * s_row[jj];
    }
    __syncthreads();
    // pivot row and pivot column
    if (tid < nb && k0 + tid != k) A[(int64_t)(k0 + tid) * m + k] = s_row[tid];
    for (int i = tid; i < m; i += blockDim.x)
      A[(int64_t)k * m + i] = (i == k) ? dinv : -A[(int64_t)k * m + i] * dinv;
    __syncthreads();
  }
}

// One thread per column outside the panel: the panel's row swaps, then X = the
// pivot rows (nb x m, row-major per matrix) and zero them in A.
__global__ void k_gj_swap_x(double *__restrict__ Aall, int m, int k0, int nb, const int32_t *__restrict__ pivall,
                            double *__restrict__ Xall) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= m) return;
  double *X = Xall + (int64_t)blockIdx.y * GJ_NB * m;
  if (j >= k0 && j < k0 + nb) {
    for (int t = 0; t < nb; ++t) X[(int64_t)t * m + j] = 0.0;
    return;
  }
  double *cj = Aall + (int64_t)blockIdx.y * m * m + (int64_t)j * m;
  const int32_t *piv = pivall + (int64_t)blockIdx.y * m;
  for (int t = 0; t < nb; ++t) {
    const int k = k0 + t, p = piv[k];
    if (p != k) {
      const double tmp = cj[k];
      cj[k] = cj[p];
      cj[p] = tmp;
    }
  }
  for (int t = 0; t < nb; ++t) {
    X[(int64_t)t * m + j] = cj[k0 + t];
    cj[k0 + t] = 0.0;
  }
}

// A[i][j] += sum_t Panel[i][t] X[t][j] on a 64 x 64 tile, columns outside the
// panel only (X is zero on panel columns, which are skipped).  256 threads, 4x4
// outputs each; the panel and X tiles staged in shared memory.
__global__ void __launch_bounds__(256) k_gj_update(double *__restrict__ Aall, int m, int k0, int nb,
                                                   const double *__restrict__ Xall) {
  __shared__ double sP[GJ_NB][GJ_T + 1];  // sP[t][i]
  __shared__ double sX[GJ_NB][GJ_T + 1];  // sX[t][j]
  double *A = Aall + (int64_t)blockIdx.z * m * m;
  const double *X = Xall + (int64_t)blockIdx.z * GJ_NB * m;
  const int i0 = blockIdx.x * GJ_T, j0 = blockIdx.y * GJ_T;
  if (j0 >= k0 && j0 + GJ_T <= k0 + nb) return;  // tile entirely inside the panel
  const int tid = threadIdx.x;
  for (int e = tid; e < nb * GJ_T; e += 256) {
    const int t = e / GJ_T, x = e % GJ_T;
    const int i = i0 + x, j = j0 + x;
    sP[t][x] = (i < m) ? A[(int64_t)(k0 + t) * m + i] : 0.0;
    sX[t][x] = (j < m) ? X[(int64_t)t * m + j] : 0.0;
  }
  __syncthreads();
  const int ti = tid % 16, tj = tid / 16;  // rows ti + 16 a, columns tj + 16 b
  double acc[4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b] = 0.0;
  for (int t = 0; t < nb; ++t) {
    double pv[4], xv[4];
#pragma unroll
    for (int a = 0; a < 4; ++a) pv[a] = sP[t][ti + 16 * a];
#pragma unroll
    for (int b = 0; b < 4; ++b) xv[b] = sX[t][tj + 16 * b];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) acc[a][b] = fma(pv[a], xv[b], acc[a][b]);
  }
#pragma unroll
  for (int b = 0; b < 4; ++b) {
    const int j = j0 + tj + 16 * b;
    if (j >= m || (j >= k0 && j < k0 + nb)) continue;
#pragma unroll
    for (int a = 0; a < 4; ++a) {
      const int i = i0 + ti + 16 * a;
      if (i < m) A[(int64_t)j * m + i] += acc[a][b];
    }
  }
}

// Column unscrambling: columns swapped (k, piv[k]) for k = m-1 .. 0, i.e.
// out[:, c] = A[:, idx[c]] with idx the reverse-order composition.
__global__ void k_gj_colidx(const int32_t *__restrict__ pivall, int m, int32_t *__restrict__ idxall) {
  if (threadIdx.x != 0) return;
  const int32_t *piv = pivall + (int64_t)blockIdx.x * m;
  int32_t *idx = idxall + (int64_t)blockIdx.x * m;
  for (int c = 0; c < m; ++c) idx[c] = c;
  for (int k = m - 1; k >= 0; --k) {
    const int p = piv[k];
    const int32_t t = idx[k];
    idx[k] = idx[p];
    idx[p] = t;
  }
}

__global__ void k_gj_unpermute(const double *__restrict__ Aall, int m, const int32_t *__restrict__ idxall,
                               double *__restrict__ outall) {
  const int64_t mm = (int64_t)m * m;
  const double *A = Aall + blockIdx.y * mm;
  const int32_t *idx = idxall + (int64_t)blockIdx.y * m;
  double *out = outall + blockIdx.y * mm;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < mm; e += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(e / m), r = (int)(e % m);
    out[e] = A[(int64_t)idx[c] * m + r];
  }
}

}  // namespace

size_t gj_scratch_doubles(int m, int batch) {
  // X panels (batch x NB x m) + tolerances (batch) + column index (batch x m int32, as doubles)
  return (size_t)batch * GJ_NB * m + (size_t)batch + ((size_t)batch * m + 1) / 2;
}

void launch_gj_inverse_batched(double *A, int m, int batch, int32_t *piv, int32_t *info, double *out,
                               double *scratch, cudaStream_t s) {
  if (batch <= 0 || m <= 0) return;
  double *X = scratch;
  double *tol = X + (size_t)batch * GJ_NB * m;
  int32_t *idx = reinterpret_cast<int32_t *>(tol + batch);
  k_gj_tol<<<batch, 1024, 0, s>>>(A, m, tol, info);
  ++g_launches;
  const int nt = (m + GJ_T - 1) / GJ_T;
  for (int k0 = 0; k0 < m; k0 += GJ_NB) {
    const int nb = std::min(GJ_NB, m - k0);
    k_gj_panel<<<batch, GJ_PTH, 0, s>>>(A, m, k0, nb, piv, info, tol);
    k_gj_swap_x<<<dim3((m + 127) / 128, batch), 128, 0, s>>>(A, m, k0, nb, piv, X);
    k_gj_update<<<dim3(nt, nt, batch), 256, 0, s>>>(A, m, k0, nb, X);
    g_launches += 3;
  }
  k_gj_colidx<<<batch, 32, 0, s>>>(piv, m, idx);
  const int64_t mm = (int64_t)m * m;
  k_gj_unpermute<<<dim3((unsigned)std::min<int64_t>((mm + 255) / 256, 4096), batch), 256, 0, s>>>(A, m, idx, out);
  g_launches += 2;
}

}  // namespace wrmg
