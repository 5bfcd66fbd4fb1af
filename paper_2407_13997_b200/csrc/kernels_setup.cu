// Setup / linearisation kernels: spatial assembly (H1), local space-time patch
// blocks (H4), batched dense LU with partial pivoting (H5), explicit inverses
// and jump propagators used by the sweep, and the coarse-level block.
#include <cfloat>

#include "internal.h"
#include "lattice.h"

namespace wrmg {
namespace {

__device__ __forceinline__ int csr_find(const int32_t *rowptr, const int32_t *col, int64_t i, int32_t j) {
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

// H1: row i of M (val) and kappa*K (val2) by summing the element matrices of
// the triangles containing node i (one thread owns the row: deterministic).
__global__ void k_assemble(int k, int nx, int ny, int Lx, int64_t nnode, double h2, double kappa,
                           const int32_t *__restrict__ rowptr, const int32_t *__restrict__ col,
                           double *__restrict__ Mv, double *__restrict__ Kv, const double *__restrict__ ref,
                           int nloc) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= nnode) return;
  int I = (int)(i % Lx), J = (int)(i / Lx);
  for (int e = rowptr[i]; e < rowptr[i + 1]; ++e) {
    Mv[e] = 0.0;
    Kv[e] = 0.0;
  }
  int ci[6], cj[6], t[6], la[6], lb[6];
  int nc = cells_of_node(k, nx, ny, I, J, ci, cj, t, la, lb);
  const double *refM = ref, *refK = ref + nloc * nloc;
  for (int c = 0; c < nc; ++c) {
    int li = loc_index(k, la[c], lb[c]);
    for (int b = 0; b <= k; ++b)
      for (int a = 0; a + b <= k; ++a) {
        int lj = loc_index(k, a, b);
        int I2, J2;
        loc_to_lattice(k, ci[c], cj[c], t[c], a, b, &I2, &J2);
        int pos = csr_find(rowptr, col, i, J2 * Lx + I2);
        Mv[pos] += h2 * refM[li * nloc + lj];
        Kv[pos] += kappa * refK[li * nloc + lj];
      }
  }
}

struct TM {
  double CE[16], Mt[16];
};

// H4: D[(a,i),(b,j)] = (C+E0)_ab M_ij + Mt_ab kappa K_ij, column-major, for the
// representative patch of each translation class; pad DoFs get identity rows.
__global__ void k_patch_blocks(const int32_t *__restrict__ rowptr, const int32_t *__restrict__ col,
                               const double *__restrict__ Mv, const double *__restrict__ Kv,
                               const int32_t *__restrict__ pnodes, const int32_t *__restrict__ rep, int mp, int nq,
                               TM tm, double *__restrict__ D) {
  const int t = blockIdx.x, m = nq * mp;
  const int32_t *nodes = pnodes + (int64_t)rep[t] * mp;
  double *Dt = D + (int64_t)t * m * m;
  for (int e = threadIdx.x; e < m * m; e += blockDim.x) {
    int rho = e % m, sig = e / m;  // column-major: e = sig*m + rho
    int a = rho / mp, i = rho % mp, b = sig / mp, j = sig % mp;
    int ni = nodes[i], nj = nodes[j];
    double v;
    if (ni < 0 || nj < 0) {
      v = (rho == sig) ? 1.0 : 0.0;
    } else {
      int pos = csr_find(rowptr, col, ni, nj);
      double mij = pos >= 0 ? Mv[pos] : 0.0, kij = pos >= 0 ? Kv[pos] : 0.0;
      v = tm.CE[a * nq + b] * mij + tm.Mt[a * nq + b] * kij;
    }
    Dt[e] = v;
  }
}

// Coarse block over all free coarse nodes (one "patch", no padding).
__global__ void k_coarse_block(const int32_t *__restrict__ rowptr, const int32_t *__restrict__ col,
                               const double *__restrict__ Mv, const double *__restrict__ Kv,
                               const int32_t *__restrict__ nodes, int mp, int nq, TM tm, double *__restrict__ D) {
  const int64_t m = (int64_t)nq * mp;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m * m; e += (int64_t)gridDim.x * blockDim.x) {
    int rho = (int)(e % m), sig = (int)(e / m);
    int a = rho / mp, i = rho % mp, b = sig / mp, j = sig % mp;
    int pos = csr_find(rowptr, col, nodes[i], nodes[j]);
    double mij = pos >= 0 ? Mv[pos] : 0.0, kij = pos >= 0 ? Kv[pos] : 0.0;
    D[e] = tm.CE[a * nq + b] * mij + tm.Mt[a * nq + b] * kij;
  }
}

// H5: right-looking LU with partial pivoting of one column-major m x m matrix
// per CTA (LAPACK dgetrf semantics: first maximum |a|, rows swapped across all
// columns, unit-lower L).  Pivot search: warp-shuffle argmax, then across warps.
// Singular (R10): |pivot| < 1e-14 * max_i sum_j |a_ij| of the input matrix.
template <bool SMEM>
__global__ void __launch_bounds__(256) k_batched_lu(double *__restrict__ Aall, int m, int32_t *__restrict__ piv,
                                                    int32_t *__restrict__ info) {
  extern __shared__ double sm[];
  __shared__ double s_val[8];
  __shared__ int s_idx[8];
  __shared__ double s_tol;
  __shared__ int s_info;
  double *g = Aall + (int64_t)blockIdx.x * m * m;
  double *A = SMEM ? sm : g;
  const int tid = threadIdx.x, nth = blockDim.x, lane = tid & 31, wid = tid >> 5, nw = nth >> 5;
  if (SMEM)
    for (int e = tid; e < m * m; e += nth) A[e] = g[e];
  __syncthreads();  // the row norms below read rows staged by other threads
  // max row norm
  double rn = 0.0;
  for (int r = tid; r < m; r += nth) {
    double s = 0.0;
    for (int c = 0; c < m; ++c) s += fabs(A[(int64_t)c * m + r]);
    rn = fmax(rn, s);
  }
  for (int o = 16; o; o >>= 1) rn = fmax(rn, __shfl_xor_sync(0xffffffffu, rn, o));
  if (lane == 0) s_val[wid] = rn;
  if (tid == 0) s_info = 0;
  __syncthreads();
  if (tid == 0) {
    double mx = 0.0;
    for (int w = 0; w < nw; ++w) mx = fmax(mx, s_val[w]);
    s_tol = 1e-14 * mx;
  }
  __syncthreads();
  for (int c = 0; c < m; ++c) {
    // argmax |A[r, c]|, r >= c, ties -> smallest r
    double bv = -1.0;
    int bi = m;
    for (int r = c + tid; r < m; r += nth) {
      double v = fabs(A[(int64_t)c * m + r]);
      if (v > bv) {
        bv = v;
        bi = r;
      }
    }
    for (int o = 16; o; o >>= 1) {
      double ov = __shfl_xor_sync(0xffffffffu, bv, o);
      int oi = __shfl_xor_sync(0xffffffffu, bi, o);
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
      s_idx[0] = ix;
      piv[(int64_t)blockIdx.x * m + c] = ix;
      if (v < s_tol && s_info == 0) s_info = c + 1;
    }
    __syncthreads();
    const int p = s_idx[0];
    if (p != c)
      for (int j = tid; j < m; j += nth) {
        double t = A[(int64_t)j * m + c];
        A[(int64_t)j * m + c] = A[(int64_t)j * m + p];
        A[(int64_t)j * m + p] = t;
      }
    __syncthreads();
    const double d = A[(int64_t)c * m + c];
    if (d != 0.0)
      for (int r = c + 1 + tid; r < m; r += nth) A[(int64_t)c * m + r] /= d;
    __syncthreads();
    const int rem = m - c - 1;
    for (int e = tid; e < rem * rem; e += nth) {
      int r = c + 1 + e % rem, j = c + 1 + e / rem;
      A[(int64_t)j * m + r] -= A[(int64_t)c * m + r] * A[(int64_t)j * m + c];
    }
    __syncthreads();
  }
  if (SMEM)
    for (int e = tid; e < m * m; e += nth) g[e] = A[e];
  if (tid == 0) info[blockIdx.x] = s_info;
}

// Inverse from the LU factors: thread t solves A x = e_t in place in column t
// of the output.  ROWMAJOR: out[rho*ld + t] (m padded rows) else out[t*m + rho].
template <bool ROWMAJOR>
__global__ void k_lu_inverse(const double *__restrict__ LUall, const int32_t *__restrict__ pivall, int m,
                             double *__restrict__ outall) {
  const double *LU = LUall + (int64_t)blockIdx.y * m * m;
  const int32_t *piv = pivall + (int64_t)blockIdx.y * m;
  double *out = outall + (int64_t)blockIdx.y * m * m;
  int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= m) return;
  auto X = [&](int r) -> double & { return ROWMAJOR ? out[(int64_t)r * m + t] : out[(int64_t)t * m + r]; };
  for (int r = 0; r < m; ++r) X(r) = (r == t) ? 1.0 : 0.0;
  for (int c = 0; c < m; ++c) {
    int p = piv[c];
    if (p != c) {
      double tmp = X(c);
      X(c) = X(p);
      X(p) = tmp;
    }
  }
  for (int c = 0; c < m; ++c) {
    double xc = X(c);
    if (xc != 0.0)
      for (int r = c + 1; r < m; ++r) X(r) -= LU[(int64_t)c * m + r] * xc;
  }
  for (int c = m - 1; c >= 0; --c) {
    double xc = X(c) / LU[(int64_t)c * m + c];
    X(c) = xc;
    for (int r = 0; r < c; ++r) X(r) -= LU[(int64_t)c * m + r] * xc;
  }
}

// Jump propagator G[rho][j] = sum_i Dinv[rho][(0,i)] M_p[i][j] (row-major, m x mp):
// the solution's response to the carried end trace y_{n-1} (E1 = e_0 e_q^T, R2).
__global__ void k_patch_G(const int32_t *__restrict__ rowptr, const int32_t *__restrict__ col,
                          const double *__restrict__ Mv, const int32_t *__restrict__ pnodes,
                          const int32_t *__restrict__ rep, int mp, int nq, const double *__restrict__ Dinv,
                          double *__restrict__ G) {
  const int t = blockIdx.x, m = nq * mp;
  const int32_t *nodes = pnodes + (int64_t)rep[t] * mp;
  const double *Di = Dinv + (int64_t)t * m * m;
  double *Gt = G + (int64_t)t * m * mp;
  for (int e = threadIdx.x; e < m * mp; e += blockDim.x) {
    int rho = e / mp, j = e % mp;
    double s = 0.0;
    if (nodes[j] >= 0)
      for (int i = 0; i < mp; ++i) {
        if (nodes[i] < 0) continue;
        int pos = csr_find(rowptr, col, nodes[i], nodes[j]);
        if (pos >= 0) s += Di[(int64_t)rho * m + i] * Mv[pos];
      }
    Gt[e] = s;
  }
}

// Coarse: GT[j*m + rho] = sum_i Dinv[rho][i] M[i][j]; Dinv column-major.
__global__ void k_coarse_G(const int32_t *__restrict__ rowptr, const int32_t *__restrict__ col,
                           const double *__restrict__ Mv, const int32_t *__restrict__ nodes, int mp, int nq,
                           const double *__restrict__ DinvT, double *__restrict__ GT, double *__restrict__ Gq) {
  const int64_t m = (int64_t)nq * mp;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m * mp; e += (int64_t)gridDim.x * blockDim.x) {
    int rho = (int)(e % m), j = (int)(e / m);
    double s = 0.0;
    for (int i = 0; i < mp; ++i) {
      int pos = csr_find(rowptr, col, nodes[i], nodes[j]);
      if (pos >= 0) s += DinvT[(int64_t)i * m + rho] * Mv[pos];
    }
    GT[e] = s;
    int a = rho / mp;
    if (a == nq - 1) Gq[(int64_t)(rho % mp) * mp + j] = s;
  }
}

TM make_tm(const Temporal &T) {
  TM tm{};
  for (int e = 0; e < T.nq * T.nq; ++e) {
    tm.CE[e] = T.CE[e];
    tm.Mt[e] = T.Mt[e];
  }
  return tm;
}

}  // namespace

void launch_assemble_spatial(const Level &L, int k, const double *ref_dev, double kappa, cudaStream_t s) {
  int nloc = (k + 1) * (k + 2) / 2;
  int blocks = (int)((L.nnode + 127) / 128);
  k_assemble<<<blocks, 128, 0, s>>>(k, L.nx, L.ny, L.Lx, L.nnode, L.h * L.h, kappa, L.A.rowptr, L.A.col, L.A.val,
                                    L.A.val2, ref_dev, nloc); ++g_launches;
}

void launch_patch_blocks(const Level &L, int nq, const Temporal &tm, cudaStream_t s) {
  k_patch_blocks<<<L.ntypes, 256, 0, s>>>(L.A.rowptr, L.A.col, L.A.val, L.A.val2, L.pnodes, L.type_rep, L.mp, nq,
                                          make_tm(tm), L.Dblk); ++g_launches;
}

void launch_batched_lu(double *A, int m, int batch, int32_t *piv, int32_t *info, cudaStream_t s) {
  if (batch <= 0) return;
  size_t bytes = (size_t)m * m * sizeof(double);
  if (bytes <= 200 * 1024) {
    smem_optin((const void *)k_batched_lu<true>, 210 * 1024);
    k_batched_lu<true><<<batch, 256, bytes, s>>>(A, m, piv, info); ++g_launches;
  } else {
    k_batched_lu<false><<<batch, 256, 0, s>>>(A, m, piv, info); ++g_launches;
  }
}

void launch_inverse_and_G(const Level &L, const double *LU, int nq, cudaStream_t s) {
  int m = nq * L.mp;
  dim3 grid((m + 127) / 128, L.ntypes);
  k_lu_inverse<true><<<grid, 128, 0, s>>>(LU, L.piv, m, L.Dinv); ++g_launches;
  k_patch_G<<<L.ntypes, 256, 0, s>>>(L.A.rowptr, L.A.col, L.A.val, L.pnodes, L.type_rep, L.mp, nq, L.Dinv, L.G); ++g_launches;
}

void launch_coarse_blocks(const Level &L, Coarse &C, int nq, const Temporal &tm, cudaStream_t s) {
  int64_t mm = (int64_t)C.m * C.m;
  int blocks = (int)std::min<int64_t>((mm + 255) / 256, 4096);
  k_coarse_block<<<blocks, 256, 0, s>>>(L.A.rowptr, L.A.col, L.A.val, L.A.val2, C.nodes, C.mp, nq, make_tm(tm),
                                        C.Dblk); ++g_launches;
}

void launch_coarse_inverse(Coarse &C, const double *LU, const Level &L, int nq, cudaStream_t s) {
  dim3 grid((C.m + 127) / 128, 1);
  k_lu_inverse<false><<<grid, 128, 0, s>>>(LU, C.piv, C.m, C.DinvT); ++g_launches;
  launch_coarse_G(C, L, nq, s);
}

void launch_coarse_G(Coarse &C, const Level &L, int nq, cudaStream_t s) {
  int64_t n = (int64_t)C.m * C.mp;
  int blocks = (int)std::min<int64_t>((n + 255) / 256, 4096);
  k_coarse_G<<<blocks, 256, 0, s>>>(L.A.rowptr, L.A.col, L.A.val, C.nodes, C.mp, nq, C.DinvT, C.GT, C.Gq); ++g_launches;
}

}  // namespace wrmg

namespace wrmg {
void launch_lu_inverse_batched(const double *LU, const int32_t *piv, int m, int batch, double *out, cudaStream_t s) {
  if (batch <= 0) return;
  dim3 grid((m + 127) / 128, batch);
  k_lu_inverse<false><<<grid, 128, 0, s>>>(LU, piv, m, out);
  ++g_launches;
}
}  // namespace wrmg
