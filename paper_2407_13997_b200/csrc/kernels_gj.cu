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

// Panel kernel: the m x nb panel (contiguous in the column-major layout) is staged
// in shared memory, eliminated there, and written back; thread 0 also records the
// panel's row interchanges as one composite map (rows dst[l] <- src[l], l < cnt)
// for the other columns.
__global__ void __launch_bounds__(GJ_PTH) k_gj_panel(double *__restrict__ Aall, int m, int k0, int nb,
                                                      int32_t *__restrict__ pivall, int32_t *__restrict__ info,
                                                      const double *__restrict__ tol, int32_t *__restrict__ rmap) {
  extern __shared__ __align__(16) double P[];  // P[jj * m + i] = A[i][k0 + jj]
  __shared__ double s_val[32];
  __shared__ int s_idx[32];
  __shared__ double s_row[GJ_NB];
  __shared__ int s_p;
  double *A = Aall + (int64_t)blockIdx.x * m * m + (int64_t)k0 * m;
  int32_t *piv = pivall + (int64_t)blockIdx.x * m;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, nw = blockDim.x >> 5;
  const int tot = m * nb;
  for (int e = tid; e < tot; e += blockDim.x) P[e] = A[e];
  __syncthreads();
  for (int t = 0; t < nb; ++t) {
    const int k = k0 + t;
    const double *pk = P + t * m;
    double bv = -1.0;
    int bi = m;
    for (int r = k + tid; r < m; r += blockDim.x) {
      const double v = fabs(pk[r]);
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
    const double d = P[t * m + p];  // pivot value (row p before the interchange)
    const double dinv = d != 0.0 ? 1.0 / d : 0.0;
    if (tid < nb) {  // interchange rows k, p of the panel; scaled pivot row
      double *cj = P + tid * m;
      const double a = cj[p];
      cj[p] = cj[k];
      cj[k] = a;
      s_row[tid] = a * dinv;
    }
    __syncthreads();
    // other rows: A[i][j] -= A[i][k] row_k[j]   (j != k in the panel)
    for (int e = tid; e < tot; e += blockDim.x) {
      const int jj = e / m, i = e - jj * m;
      if (i == k || jj == t) continue;
      P[e] = fma(-pk[i], s_row[jj], P[e]);
    }
    __syncthreads();
    if (tid < nb && tid != t) P[tid * m + k] = s_row[tid];
    for (int i = tid; i < m; i += blockDim.x) P[t * m + i] = (i == k) ? dinv : -pk[i] * dinv;
    __syncthreads();
  }
  for (int e = tid; e < tot; e += blockDim.x) A[e] = P[e];
  if (tid == 0) {  // composite row map of the panel's interchanges
    int32_t *mp = rmap + (int64_t)blockIdx.x * (4 * GJ_NB + 1);
    int dst[2 * GJ_NB], src[2 * GJ_NB], cnt = 0;
    auto slot = [&](int r) {
      for (int l = 0; l < cnt; ++l)
        if (dst[l] == r) return l;
      dst[cnt] = r;
      src[cnt] = r;
      return cnt++;
    };
    for (int t = 0; t < nb; ++t) {
      const int k = k0 + t, pr = piv[k];
      if (pr == k) continue;
      const int a = slot(k), b = slot(pr);
      const int tmp = src[a];
      src[a] = src[b];
      src[b] = tmp;
    }
    mp[0] = cnt;
    for (int l = 0; l < cnt; ++l) {
      mp[1 + 2 * l] = dst[l];
      mp[2 + 2 * l] = src[l];
    }
  }
}

// Warp per column outside the panel: the panel's row interchanges (composite map,
// all loads before any store), then X = the pivot rows (nb x m per matrix), zeroed in A.
__global__ void k_gj_swap_x(double *__restrict__ Aall, int m, int k0, int nb, const int32_t *__restrict__ rmap,
                            double *__restrict__ Xall) {
  const int j = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (j >= m) return;
  double *X = Xall + (int64_t)blockIdx.y * GJ_NB * m;
  if (j >= k0 && j < k0 + nb) {
    for (int t = lane; t < nb; t += 32) X[(int64_t)t * m + j] = 0.0;
    return;
  }
  double *cj = Aall + (int64_t)blockIdx.y * m * m + (int64_t)j * m;
  const int32_t *mp = rmap + (int64_t)blockIdx.y * (4 * GJ_NB + 1);
  const int cnt = mp[0];
  double v[2];
  int dr[2];
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int l = lane + 32 * h;
    dr[h] = l < cnt ? mp[1 + 2 * l] : -1;
    v[h] = l < cnt ? cj[mp[2 + 2 * l]] : 0.0;
  }
  __syncwarp();
#pragma unroll
  for (int h = 0; h < 2; ++h)
    if (dr[h] >= 0) cj[dr[h]] = v[h];
  __syncwarp();
  for (int t = lane; t < nb; t += 32) {
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

// grid (m columns, batch): out[:, c] = A[:, idx[c]]
__global__ void k_gj_unpermute(const double *__restrict__ Aall, int m, const int32_t *__restrict__ idxall,
                               double *__restrict__ outall) {
  const int64_t mm = (int64_t)m * m;
  const int c = blockIdx.x;
  const int32_t *idx = idxall + (int64_t)blockIdx.y * m;
  const double *src = Aall + blockIdx.y * mm + (int64_t)idx[c] * m;
  double *dst = outall + blockIdx.y * mm + (int64_t)c * m;
  for (int r = threadIdx.x; r < m; r += blockDim.x) dst[r] = src[r];
}

}  // namespace

size_t gj_scratch_doubles(int m, int batch) {
  // X panels (batch x NB x m) + tolerances (batch) + column index (batch x m int32) + row maps
  // (batch x (4 NB + 1) int32), the int32 parts counted in doubles
  return (size_t)batch * GJ_NB * m + (size_t)batch + ((size_t)batch * m + 1) / 2 +
         ((size_t)batch * (4 * GJ_NB + 1) + 1) / 2 + 1;
}

void launch_gj_inverse_batched(double *A, int m, int batch, int32_t *piv, int32_t *info, double *out,
                               double *scratch, cudaStream_t s) {
  if (batch <= 0 || m <= 0) return;
  double *X = scratch;
  double *tol = X + (size_t)batch * GJ_NB * m;
  int32_t *idx = reinterpret_cast<int32_t *>(tol + batch);
  int32_t *rmap = idx + (size_t)batch * m;
  k_gj_tol<<<batch, 1024, 0, s>>>(A, m, tol, info);
  ++g_launches;
  // panel width: the m x nb panel must fit in shared memory
  const int NBP = std::max(1, std::min(GJ_NB, (int)((220 * 1024) / (sizeof(double) * (size_t)m))));
  smem_optin((const void *)k_gj_panel, 221 * 1024);
  const int nt = (m + GJ_T - 1) / GJ_T;
  for (int k0 = 0; k0 < m; k0 += NBP) {
    const int nb = std::min(NBP, m - k0);
    k_gj_panel<<<batch, GJ_PTH, (size_t)m * nb * sizeof(double), s>>>(A, m, k0, nb, piv, info, tol, rmap);
    k_gj_swap_x<<<dim3((m + 7) / 8, batch), 256, 0, s>>>(A, m, k0, nb, rmap, X);
    k_gj_update<<<dim3(nt, nt, batch), 256, 0, s>>>(A, m, k0, nb, X);
    g_launches += 3;
  }
  k_gj_colidx<<<batch, 32, 0, s>>>(piv, m, idx);
  k_gj_unpermute<<<dim3((unsigned)m, batch), 256, 0, s>>>(A, m, idx, out);
  g_launches += 2;
}

}  // namespace wrmg
