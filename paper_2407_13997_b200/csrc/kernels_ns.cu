// Navier-Stokes hot-path kernels (Taylor-Hood P_{k+1}-P_k x DG(q), eq. nsfem,
// PAPER.md:245-271; Newton linearisation DESIGN.md R18):
//   H1  spatial assembly: linear sid CSR values M2 (velocity mass) and KG (vector
//       Laplacian + divergence blocks, R17), convection R N(w_{n,c}) per (slab,
//       temporal node) on the velocity-velocity entries;
//   H4+H5 per-(patch, slab) Vanka+star block D_{p,n} assembled in shared memory and
//       inverted in place by Gauss-Jordan with partial pivoting (the pivot rows of
//       LAPACK dgetrf, R10), written row-major for the sweep;
//   H6  space-time residual, warp per sid row, lanes over slabs;
//   H7+H8 forward time sweep: per patch, D_{p,n}^{-1} streamed slab by slab with
//       TMA bulk copies into a double buffer, jump carried from slab n-1,
//       weighted additive scatter with FP64 atomics (R9, R11);
//   H11 coarse blocks with the pinned pressure DoF (R19) and the time-marching solve;
//   H15 pressure mean projection per (slab, temporal node) (R19);
//   state injection to coarse levels (R13).
#include <cooperative_groups.h>

#include <algorithm>
#include <cfloat>

#include "lattice.h"
#include "ns_kernels.h"

namespace wrmg {
namespace {

__device__ __forceinline__ int csr_find_ns(const int32_t *rowptr, const int32_t *col, int64_t i, int32_t j) {
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

// ------------------------------------------------------------------ H1 linear
// Row r of M2 (val) and K2 + G-blocks (val2).  Triangle t maps x = v0 + s h xi,
// s = +1 (t = 0) / -1 (t = 1): M = h^2 Mh, K = Kh, G = s h Gh, To = s h Th.
__global__ void k_ns_assemble_linear(NSGeom g, const int32_t *__restrict__ rowptr, const int32_t *__restrict__ col,
                                     double *__restrict__ Mv, double *__restrict__ KGv, const double *__restrict__ ref) {
  const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (r >= g.ns) return;
  const int nu = g.nu, np = g.np;
  const double *Mh = ref, *Kh = ref + nu * nu, *Gh = ref + 2 * nu * nu;
  for (int e = rowptr[r]; e < rowptr[r + 1]; ++e) {
    Mv[e] = 0.0;
    KGv[e] = 0.0;
  }
  int ci[6], cj[6], t[6], la[6], lb[6];
  if (r < 2 * g.Lu) {
    const int d = (int)(r / g.Lu);
    const int64_t i = r - d * g.Lu;
    const int I = (int)(i % g.Lux), J = (int)(i / g.Lux);
    const int nc = cells_of_node(g.ku, g.nx, g.ny, I, J, ci, cj, t, la, lb);
    for (int c = 0; c < nc; ++c) {
      const double s = t[c] == 0 ? 1.0 : -1.0;
      const int li = loc_index(g.ku, la[c], lb[c]);
      for (int b = 0; b <= g.ku; ++b)
        for (int a = 0; a + b <= g.ku; ++a) {
          int I2, J2;
          loc_to_lattice(g.ku, ci[c], cj[c], t[c], a, b, &I2, &J2);
          const int lj = loc_index(g.ku, a, b);
          const int pos = csr_find_ns(rowptr, col, r, (int32_t)(d * g.Lu + (int64_t)J2 * g.Lux + I2));
          Mv[pos] += g.h * g.h * Mh[li * nu + lj];
          KGv[pos] += Kh[li * nu + lj];
        }
      for (int b = 0; b <= g.kp; ++b)
        for (int a = 0; a + b <= g.kp; ++a) {
          int I2, J2;
          loc_to_lattice(g.kp, ci[c], cj[c], t[c], a, b, &I2, &J2);
          const int lp = loc_index(g.kp, a, b);
          const int pos = csr_find_ns(rowptr, col, r, (int32_t)(2 * g.Lu + (int64_t)J2 * g.Lpx + I2));
          KGv[pos] += s * g.h * Gh[(d * nu + li) * np + lp];
        }
    }
  } else {
    const int64_t j = r - 2 * g.Lu;
    const int Ip = (int)(j % g.Lpx), Jp = (int)(j / g.Lpx);
    const int nc = cells_of_node(g.kp, g.nx, g.ny, Ip, Jp, ci, cj, t, la, lb);
    for (int c = 0; c < nc; ++c) {
      const double s = t[c] == 0 ? 1.0 : -1.0;
      const int lp = loc_index(g.kp, la[c], lb[c]);
      for (int b = 0; b <= g.ku; ++b)
        for (int a = 0; a + b <= g.ku; ++a) {
          int I2, J2;
          loc_to_lattice(g.ku, ci[c], cj[c], t[c], a, b, &I2, &J2);
          const int lj = loc_index(g.ku, a, b);
          const int64_t node = (int64_t)J2 * g.Lux + I2;
          for (int d = 0; d < 2; ++d) {
            const int pos = csr_find_ns(rowptr, col, r, (int32_t)(d * g.Lu + node));
            KGv[pos] += s * g.h * Gh[(d * nu + lj) * np + lp];
          }
        }
    }
  }
}

// --------------------------------------------------------------- H1 convection
// conv[e][t] = R N(w_t) on the velocity-velocity entries e of the sid CSR, t =
// n (q+1) + c.  N(w) = O(w) (+ Q(w) for the Newton Jacobian, R18):
//   O[(d,i),(d,j)]  = sum_l sum_d2 w[l,d2] int v_i v_l d_d2 v_j
//   Q[(d,i),(d2,j)] = sum_l w[l,d] int v_i v_j d_d2 v_l.
// Thread = (velocity node i, t): owns column t of rows (0,i) and (1,i).
__global__ void __launch_bounds__(256) k_ns_assemble_conv(NSGeom g, int64_t NT, double R, int newton,
                                                          const int32_t *__restrict__ rowptr,
                                                          const int32_t *__restrict__ col,
                                                          const int32_t *__restrict__ vvptr,
                                                          const double *__restrict__ W, double *__restrict__ conv,
                                                          const double *__restrict__ Th_g) {
  extern __shared__ double Th[];
  const int nu = g.nu;
  for (int e = threadIdx.x; e < 2 * nu * nu * nu; e += blockDim.x) Th[e] = Th_g[e];
  __syncthreads();
  const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (idx >= g.Lu * NT) return;
  const int64_t i = idx / NT, tt = idx - i * NT;
  const int64_t r0 = i, r1 = g.Lu + i;
  for (int e = vvptr[r0]; e < vvptr[r0 + 1]; ++e) conv[(int64_t)e * NT + tt] = 0.0;
  for (int e = vvptr[r1]; e < vvptr[r1 + 1]; ++e) conv[(int64_t)e * NT + tt] = 0.0;
  if (W == nullptr) return;
  const int I = (int)(i % g.Lux), J = (int)(i / g.Lux);
  int ci[6], cj[6], t[6], la[6], lb[6];
  const int nc = cells_of_node(g.ku, g.nx, g.ny, I, J, ci, cj, t, la, lb);
  for (int c = 0; c < nc; ++c) {
    const double sh = (t[c] == 0 ? 1.0 : -1.0) * g.h * R;
    const int li = loc_index(g.ku, la[c], lb[c]);
    double w[kMaxLocU][2];
    int64_t node[kMaxLocU];
    for (int b = 0; b <= g.ku; ++b)
      for (int a = 0; a + b <= g.ku; ++a) {
        int I2, J2;
        loc_to_lattice(g.ku, ci[c], cj[c], t[c], a, b, &I2, &J2);
        const int l = loc_index(g.ku, a, b);
        node[l] = (int64_t)J2 * g.Lux + I2;
        w[l][0] = W[node[l] * NT + tt];
        w[l][1] = W[(g.Lu + node[l]) * NT + tt];
      }
    for (int lj = 0; lj < nu; ++lj) {
      double O = 0.0, Q00 = 0.0, Q01 = 0.0, Q10 = 0.0, Q11 = 0.0;
      for (int l = 0; l < nu; ++l) {
        O += w[l][0] * Th[((0 * nu + li) * nu + l) * nu + lj] + w[l][1] * Th[((1 * nu + li) * nu + l) * nu + lj];
        if (newton) {
          const double t0 = Th[((0 * nu + li) * nu + lj) * nu + l], t1 = Th[((1 * nu + li) * nu + lj) * nu + l];
          Q00 += w[l][0] * t0;
          Q01 += w[l][0] * t1;
          Q10 += w[l][1] * t0;
          Q11 += w[l][1] * t1;
        }
      }
      const int p00 = csr_find_ns(rowptr, col, r0, (int32_t)node[lj]);
      const int p01 = csr_find_ns(rowptr, col, r0, (int32_t)(g.Lu + node[lj]));
      const int p10 = csr_find_ns(rowptr, col, r1, (int32_t)node[lj]);
      const int p11 = csr_find_ns(rowptr, col, r1, (int32_t)(g.Lu + node[lj]));
      conv[(int64_t)(vvptr[r0] + p00 - rowptr[r0]) * NT + tt] += sh * (O + Q00);
      conv[(int64_t)(vvptr[r1] + p11 - rowptr[r1]) * NT + tt] += sh * (O + Q11);
      if (newton) {
        conv[(int64_t)(vvptr[r0] + p01 - rowptr[r0]) * NT + tt] += sh * Q01;
        conv[(int64_t)(vvptr[r1] + p10 - rowptr[r1]) * NT + tt] += sh * Q10;
      }
    }
  }
}

// State on the next coarser level by nodal sampling (R13): coarse node (I, J) is
// fine node (2I, 2J) on both lattices.
__global__ void k_ns_inject(NSGeom c, NSGeom f, int64_t NT, const double *__restrict__ Wf, double *__restrict__ Wc,
                            NSInjMap m) {
  const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (idx >= c.ns * NT) return;
  const int64_t s = idx / NT, tt = idx - s * NT;
  int64_t fs;
  int If;
  bool ok;
  if (s < 2 * c.Lu) {
    const int d = (int)(s / c.Lu);
    const int64_t i = s - d * c.Lu;
    const int I = (int)(i % c.Lux), J = (int)(i / c.Lux);
    If = 2 * I + m.du;
    ok = If >= m.fu0 && If <= m.fu1;
    fs = d * f.Lu + (int64_t)(2 * J) * f.Lux + If;
  } else {
    const int64_t j = s - 2 * c.Lu;
    const int I = (int)(j % c.Lpx), J = (int)(j / c.Lpx);
    If = 2 * I + m.dp;
    ok = If >= m.fp0 && If <= m.fp1;
    fs = 2 * f.Lu + (int64_t)(2 * J) * f.Lpx + If;
  }
  Wc[idx] = ok ? Wf[fs * NT + tt] : 0.0;
}

// Column sums over the lattice columns [c0, c0 + nc) of a (Ly, Lx, NT) field: one
// partial per block of lattice rows (strip pressure projection, owned columns).
__global__ void k_colsum_cols(const double *__restrict__ P, int Lx, int Ly, int c0, int nc, int64_t NT, int rpb,
                              double *__restrict__ partial) {
  const int J0 = blockIdx.x * rpb, J1 = min(Ly, J0 + rpb);
  for (int64_t t = threadIdx.x; t < NT; t += blockDim.x) {
    double acc = 0.0;
    for (int J = J0; J < J1; ++J)
      for (int c = 0; c < nc; ++c) acc += P[((int64_t)J * Lx + c0 + c) * NT + t];
    partial[blockIdx.x * NT + t] = acc;
  }
}

// ------------------------------------------------------------------ H6 residual
// r = b - A u:  (A u)_{n,a} = sum_e [(C+E0)_ab M2_e + Mt_ab KG_e] u_{col,n,b}
//   - [a = 0] M2_e u_{col,n-1,q}  + sum_{e in vv} sum_{b,c} T_abc conv_{e,n,c} u_{col,n,b}
// constrained rows r = b - u (R5).  b == NULL: r = A u (constrained rows r = u).
template <int NQ>
__global__ void __launch_bounds__(256) k_ns_residual(int64_t ns, int N, const int32_t *__restrict__ rowptr,
                                                     const int32_t *__restrict__ col, const double *__restrict__ Mv,
                                                     const double *__restrict__ KGv, int64_t nvrow,
                                                     const int32_t *__restrict__ vvptr,
                                                     const double *__restrict__ conv, const uint8_t *__restrict__ con,
                                                     const double *__restrict__ u, const double *__restrict__ b,
                                                     double *__restrict__ r, NSTime tm) {
  const int64_t row = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= ns) return;
  const int64_t NT = (int64_t)N * NQ;
  const int e0 = rowptr[row], e1 = rowptr[row + 1];
  const int nvv = row < nvrow ? vvptr[row + 1] - vvptr[row] : 0;
  const int vb = row < nvrow ? vvptr[row] : 0;
  const bool cr = con[row] != 0;
  for (int n = lane; n < N; n += 32) {
    const int64_t base = row * NT + (int64_t)n * NQ;
    double acc[NQ];
    if (cr) {
#pragma unroll
      for (int a = 0; a < NQ; ++a) r[base + a] = b ? b[base + a] - u[base + a] : u[base + a];
      continue;
    }
#pragma unroll
    for (int a = 0; a < NQ; ++a) acc[a] = 0.0;
    // entries in batches of U with every load of a batch issued before its FMAs
    // (velocity-velocity entries first: they carry the convection values)
    constexpr int U = 4;
    auto batch = [&](int e, int cnt, bool hasconv) {
      int64_t cb[U];
      double mv[U], kg[U], ub[U][NQ], um[U], w[U][NQ];
#pragma unroll
      for (int k = 0; k < U; ++k) {
        const int ek = k < cnt ? e + k : e;
        cb[k] = (int64_t)__ldg(col + ek) * NT + (int64_t)n * NQ;
        mv[k] = k < cnt ? __ldg(Mv + ek) : 0.0;
        kg[k] = k < cnt ? __ldg(KGv + ek) : 0.0;
      }
#pragma unroll
      for (int k = 0; k < U; ++k) {
        if constexpr (NQ == 2) {  // DG1: the slab's two values as one 16-byte load (NT even, offsets even)
          const double2 uv = __ldg(reinterpret_cast<const double2 *>(u + cb[k]));
          ub[k][0] = uv.x;
          ub[k][1 % NQ] = uv.y;
        } else {
#pragma unroll
          for (int bb = 0; bb < NQ; ++bb) ub[k][bb] = __ldg(u + cb[k] + bb);
        }
        um[k] = n > 0 ? __ldg(u + cb[k] - 1) : 0.0;
        if (hasconv) {
          const double *cv = conv + (int64_t)(vb + (k < cnt ? e + k : e) - e0) * NT + (int64_t)n * NQ;
          if constexpr (NQ == 2) {
            const double2 cw = k < cnt ? __ldg(reinterpret_cast<const double2 *>(cv)) : make_double2(0.0, 0.0);
            w[k][0] = cw.x;
            w[k][1 % NQ] = cw.y;
          } else {
#pragma unroll
            for (int c = 0; c < NQ; ++c) w[k][c] = k < cnt ? __ldg(cv + c) : 0.0;
          }
        }
      }
#pragma unroll
      for (int k = 0; k < U; ++k) {
#pragma unroll
        for (int a = 0; a < NQ; ++a)
#pragma unroll
          for (int bb = 0; bb < NQ; ++bb)
            acc[a] = fma(tm.CE[a * NQ + bb] * mv[k] + tm.Mt[a * NQ + bb] * kg[k], ub[k][bb], acc[a]);
        acc[0] = fma(-mv[k], um[k], acc[0]);
        if (hasconv)
#pragma unroll
          for (int a = 0; a < NQ; ++a)
#pragma unroll
            for (int bb = 0; bb < NQ; ++bb) {
              double tw = 0.0;
#pragma unroll
              for (int c = 0; c < NQ; ++c) tw = fma(tm.T[(a * NQ + bb) * NQ + c], w[k][c], tw);
              acc[a] = fma(tw, ub[k][bb], acc[a]);
            }
      }
    };
    const int ev1 = e0 + nvv;
    for (int e = e0; e < ev1; e += U) batch(e, min(U, ev1 - e), true);
    for (int e = ev1; e < e1; e += U) batch(e, min(U, e1 - e), false);
    if constexpr (NQ == 2) {
      double2 o = make_double2(acc[0], acc[1 % NQ]);
      if (b) {
        const double2 bv = *reinterpret_cast<const double2 *>(b + base);
        o = make_double2(bv.x - o.x, bv.y - o.y);
      }
      *reinterpret_cast<double2 *>(r + base) = o;
    } else {
#pragma unroll
      for (int a = 0; a < NQ; ++a) r[base + a] = b ? b[base + a] - acc[a] : acc[a];
    }
  }
}

// Per patch, the CSR positions of every (i, j) node pair of D_p (the sparsity is
// the same for every slab and linearisation): ppos = entry of the sid CSR or -1,
// pvv = the pair's index in the convection storage or -1 (pressure rows / columns).
__global__ void k_ns_patch_pos(int mp, const int32_t *__restrict__ pnodes, const int32_t *__restrict__ rowptr,
                               const int32_t *__restrict__ col, int64_t nvrow, const int32_t *__restrict__ vvptr,
                               int32_t *__restrict__ ppos, int32_t *__restrict__ pvv) {
  const int64_t p = blockIdx.x;
  for (int e = threadIdx.x; e < mp * mp; e += blockDim.x) {
    const int i = e / mp, j = e - i * mp;
    const int si = pnodes[p * mp + i], sj = pnodes[p * mp + j];
    int pos = -1, vv = -1;
    if (si >= 0 && sj >= 0) {
      pos = csr_find_ns(rowptr, col, si, sj);
      if (pos >= 0 && si < nvrow) {
        const int ev = pos - rowptr[si];
        if (ev < vvptr[si + 1] - vvptr[si]) vv = vvptr[si] + ev;
      }
    }
    ppos[p * mp * mp + e] = pos;
    pvv[p * mp * mp + e] = vv;
  }
}

// Block value from the precomputed pair tables (no searches): the same value as block_entry.
template <int NQ>
__device__ __forceinline__ double block_entry_tab(int pos, int vv, const double *__restrict__ Mv,
                                                  const double *__restrict__ KGv, const double *__restrict__ conv,
                                                  int64_t NT, int n, const NSTime &tm, int a, int bb) {
  if (pos < 0) return 0.0;
  double v = tm.CE[a * NQ + bb] * __ldg(Mv + pos) + tm.Mt[a * NQ + bb] * __ldg(KGv + pos);
  if (vv >= 0) {
    const double *cv = conv + (int64_t)vv * NT + (int64_t)n * NQ;
#pragma unroll
    for (int c = 0; c < NQ; ++c) v = fma(tm.T[(a * NQ + bb) * NQ + c], __ldg(cv + c), v);
  }
  return v;
}

// ------------------------------------------------------- H4 + H5 block inverse
// Block value D[(i,a),(j,b)] of D_{p,n} = R_p A_nn R_p^T (R9) for sids si, sj.
template <int NQ>
__device__ __forceinline__ double block_entry(const int32_t *__restrict__ rowptr, const int32_t *__restrict__ col,
                                              const double *__restrict__ Mv, const double *__restrict__ KGv,
                                              int64_t nvrow, const int32_t *__restrict__ vvptr,
                                              const double *__restrict__ conv, int64_t NT, int n, const NSTime &tm,
                                              int si, int sj, int a, int bb) {
  const int pos = csr_find_ns(rowptr, col, si, sj);
  if (pos < 0) return 0.0;
  double v = tm.CE[a * NQ + bb] * Mv[pos] + tm.Mt[a * NQ + bb] * KGv[pos];
  if (si < nvrow) {
    const int ev = pos - rowptr[si];
    if (ev < vvptr[si + 1] - vvptr[si]) {
      const double *cv = conv + (int64_t)(vvptr[si] + ev) * NT + (int64_t)n * NQ;
#pragma unroll
      for (int c = 0; c < NQ; ++c) v = fma(tm.T[(a * NQ + bb) * NQ + c], cv[c], v);
    }
  }
  return v;
}

// In-place blocked Gauss-Jordan inverse of the row-major m x m matrix A in shared
// memory with partial pivoting (first maximum |a| at or below the diagonal: the
// pivot rows LAPACK dgetrf picks, R10).  Panels of GJB columns: (1) Gauss-Jordan on
// the panel columns with whole-row interchanges; the panel becomes
// [P11^{-1}; -A_O P11^{-1}] (pivot rows / other rows); (2) X = the pivot rows of the
// other columns; (3) rank-GJB update A[:, j] = [0; A_O[:, j]] + Panel X[:, j] by 4x4
// register tiles (the 2 m^3 flops; shared-memory traffic / GJB of the column-at-a-
// time form).  The row interchanges are undone as an output column permutation:
// idx[c] = the column of A holding column c of the inverse.  Returns 0 or 1 + the
// first column with |pivot| < tol.
constexpr int GJB = 8;
// X: GJB x m (or, gj_invert_smem_lr, the pivot rows in B-fragment order: 64 per tile column)
__host__ __device__ constexpr size_t ns_factor_xdoubles(int m) {
  return (size_t)GJB * m > (size_t)64 * ((m + 7) / 8) ? (size_t)GJB * m : (size_t)64 * ((m + 7) / 8);
}
// doubles of shared memory per block in k_ns_factor_warp: A, X, and the int arrays (piv, idx, nodes)
__host__ __device__ constexpr size_t ns_factor_warp_doubles(int m, int mp) {
  return (size_t)m * m + (size_t)GJB * m + ((size_t)(2 * m + mp) + 1) / 2 + 2;
}
__device__ __forceinline__ void dmma_ns(double &c0, double &c1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(c0), "+d"(c1)
      : "d"(a), "d"(b));
}
__device__ int gj_invert_smem(double *A, int m, double tol, double *X, int *piv, int *idx) {
  __shared__ double s_val[32], s_sv[32];
  __shared__ int s_idx[32];
  __shared__ int s_info;
  const int tid = threadIdx.x, nth = blockDim.x, lane = tid & 31, wid = tid >> 5, nw = nth >> 5;
  if (tid == 0) s_info = 0;
  __syncthreads();
  for (int k0 = 0; k0 < m; k0 += GJB) {
    const int nb = min(GJB, m - k0), k1 = k0 + nb;
    for (int c = k0; c < k1; ++c) {
      // (1) argmax |A[r][c]|, r >= c (first maximum), with its signed value
      double bv = -1.0, bs = 0.0;
      int bi = m;
      for (int r = c + tid; r < m; r += nth) {
        const double sv = A[r * m + c], v = fabs(sv);
        if (v > bv) {
          bv = v;
          bs = sv;
          bi = r;
        }
      }
      for (int o = 16; o; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
        const double os = __shfl_xor_sync(0xffffffffu, bs, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ov > bv || (ov == bv && oi < bi)) {
          bv = ov;
          bs = os;
          bi = oi;
        }
      }
      if (lane == 0) {
        s_val[wid] = bv;
        s_sv[wid] = bs;
        s_idx[wid] = bi;
      }
      __syncthreads();
      // (2) every thread combines the warp maxima; whole-row interchange c <-> p, row c
      // scaled on the panel columns
      double v = s_val[0], pv = s_sv[0];
      int p = s_idx[0];
      for (int w = 1; w < nw; ++w)
        if (s_val[w] > v || (s_val[w] == v && s_idx[w] < p)) {
          v = s_val[w];
          pv = s_sv[w];
          p = s_idx[w];
        }
      if (tid == 0) {
        piv[c] = p;
        if (!(v >= tol) && s_info == 0) s_info = c + 1;
      }
      const double pinv = pv != 0.0 ? 1.0 / pv : 0.0;
      for (int j = tid; j < m; j += nth) {
        const double t1 = A[c * m + j], t2 = A[p * m + j];
        A[p * m + j] = t1;
        A[c * m + j] = (j >= k0 && j < k1) ? ((j == c) ? pinv : t2 * pinv) : t2;
      }
      __syncthreads();
      // (3) thread per row: panel rank-1 step and the pivot column, -f_r / pivot
      for (int r = tid; r < m; r += nth) {
        if (r == c) continue;
        const double fr = A[r * m + c];
        for (int j = k0; j < k1; ++j)
          if (j != c) A[r * m + j] = fma(-fr, A[c * m + j], A[r * m + j]);
        A[r * m + c] = -fr * pinv;
      }
      __syncthreads();
    }
    // X = pivot rows of the other columns
    for (int e = tid; e < nb * m; e += nth) {
      const int t = e / m, j = e - t * m;
      X[e] = (j >= k0 && j < k1) ? 0.0 : A[(k0 + t) * m + j];
    }
    __syncthreads();
    // A[:, j] = [0 on pivot rows; A] + Panel X   (columns outside the panel), on the
    // FP64 tensor cores: warp item = one 8 x 8 output tile, two mma.m8n8k4 (k = the
    // 8 panel columns).  Fragments (tools/dmma_layout.cu): a = P[l>>2][l&3],
    // b = X[l&3][l>>2], c[e] = C[l>>2][2(l&3)+e]; the panel is exactly tile column k0/8.
    {
      const int nt8 = (m + 7) / 8, pt = k0 / 8;
      const int lr = lane >> 2, lc = lane & 3;
      for (int it = wid; it < nt8 * nt8; it += nw) {
        const int tr = it / nt8, tc = it - tr * nt8;
        if (tc == pt) continue;
        const int R = tr * 8 + lr;
        const bool rok = R < m, rpiv = R >= k0 && R < k1;
        double c[2];
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int J = tc * 8 + 2 * lc + e;
          c[e] = (rok && !rpiv && J < m) ? A[R * m + J] : 0.0;
        }
        const int Jb = tc * 8 + lr;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int t = 4 * h + lc;
          const double a = (rok && t < nb) ? A[R * m + k0 + t] : 0.0;
          const double b = (t < nb && Jb < m) ? X[t * m + Jb] : 0.0;
          dmma_ns(c[0], c[1], a, b);
        }
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int J = tc * 8 + 2 * lc + e;
          if (rok && J < m) A[R * m + J] = c[e];
        }
      }
    }
    __syncthreads();
  }
  // (P A)^{-1} = A^{-1} P^T: columns interchanged (c, piv[c]) for c = m-1 .. 0
  if (tid == 0) {
    for (int c = 0; c < m; ++c) idx[c] = c;
    for (int c = m - 1; c >= 0; --c) {
      const int p = piv[c], t = idx[c];
      idx[c] = idx[p];
      idx[p] = t;
    }
  }
  __syncthreads();
  return s_info;
}

// Same elimination (same pivots, same operations per entry) with the panel columns
// factored by warp 0 alone in registers: lane l holds rows l, l + 32, ... (RPL rows)
// of the GJB panel columns; the pivot search is a warp argmax (first maximum |a|,
// lowest row on ties: R10), the pivot and displaced rows move by shuffles, the rank-1
// panel updates are lane-local FMAs.  The row interchanges reach the other columns
// afterwards (in pivot order, one thread per column), then the DMMA rank-GJB update
// as in gj_invert_smem.  Three CTA barriers per panel instead of three per column.
template <int RPL>
__device__ int gj_invert_smem_wp(double *A, int m, double tol, double *X, int *piv, int *idx) {
  __shared__ int s_info;
  const int tid = threadIdx.x, nth = blockDim.x, lane = tid & 31, wid = tid >> 5, nw = nth >> 5;
  if (tid == 0) s_info = 0;
  __syncthreads();
  for (int k0 = 0; k0 < m; k0 += GJB) {
    const int nb = min(GJB, m - k0), k1 = k0 + nb;
    if (wid == 0) {
      double P[RPL][GJB];
#pragma unroll
      for (int s = 0; s < RPL; ++s) {
        const int r = lane + 32 * s;
#pragma unroll
        for (int t = 0; t < GJB; ++t) P[s][t] = (r < m && t < nb) ? A[r * m + k0 + t] : 0.0;
      }
      int info = 0;
#pragma unroll
      for (int tc = 0; tc < GJB; ++tc) {
        if (tc >= nb) break;
        const int c = k0 + tc;
        // (1) argmax |P[r][tc]| over rows r >= c: first maximum, lowest row
        double bv = -1.0;
        int bi = m;
#pragma unroll
        for (int s = 0; s < RPL; ++s) {
          const int r = lane + 32 * s;
          const double v = fabs(P[s][tc]);
          if (r >= c && r < m && v > bv) {
            bv = v;
            bi = r;
          }
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) {
          const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
          const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
          if (ov > bv || (ov == bv && oi < bi)) {
            bv = ov;
            bi = oi;
          }
        }
        if (!(bv >= tol) && info == 0) info = c + 1;
        // (2) pivot row and row c (the rows to interchange) to every lane
        const int sp = bi >> 5, lp = bi & 31, sc = c >> 5, lc = c & 31;
        double prow[GJB], crow[GJB];
#pragma unroll
        for (int t = 0; t < GJB; ++t) {
          double vp = 0.0, vc = 0.0;
#pragma unroll
          for (int s = 0; s < RPL; ++s) {
            vp = (s == sp) ? P[s][t] : vp;
            vc = (s == sc) ? P[s][t] : vc;
          }
          prow[t] = __shfl_sync(0xffffffffu, vp, lp);
          crow[t] = __shfl_sync(0xffffffffu, vc, lc);
        }
        const double pv = prow[tc];
        const double pinv = pv != 0.0 ? 1.0 / pv : 0.0;
        double newc[GJB];  // pivot row after scaling (panel columns); column tc holds 1 / pivot
#pragma unroll
        for (int t = 0; t < GJB; ++t) newc[t] = (t == tc) ? pinv : prow[t] * pinv;
        // (3) interchange, scale, rank-1 update of the panel rows
#pragma unroll
        for (int s = 0; s < RPL; ++s) {
          const int r = lane + 32 * s;
          if (r == bi && bi != c) {
#pragma unroll
            for (int t = 0; t < GJB; ++t) P[s][t] = crow[t];
          }
          if (r == c) {
#pragma unroll
            for (int t = 0; t < GJB; ++t) P[s][t] = newc[t];
          } else {
            const double fr = P[s][tc];
#pragma unroll
            for (int t = 0; t < GJB; ++t)
              if (t != tc) P[s][t] = fma(-fr, newc[t], P[s][t]);
            P[s][tc] = -fr * pinv;
          }
        }
        if (lane == 0) piv[c] = bi;
      }
#pragma unroll
      for (int s = 0; s < RPL; ++s) {
        const int r = lane + 32 * s;
        if (r < m)
#pragma unroll
          for (int t = 0; t < GJB; ++t)
            if (t < nb) A[r * m + k0 + t] = P[s][t];
      }
      if (lane == 0 && info && s_info == 0) s_info = info;
    }
    __syncthreads();
    // the panel's row interchanges on the other columns (pivot order), then X = pivot rows
    for (int j = tid; j < m; j += nth) {
      if (j >= k0 && j < k1) continue;
      for (int c = k0; c < k1; ++c) {
        const int p = piv[c];
        if (p != c) {
          const double t1 = A[c * m + j];
          A[c * m + j] = A[p * m + j];
          A[p * m + j] = t1;
        }
      }
      for (int t = 0; t < nb; ++t) X[t * m + j] = A[(k0 + t) * m + j];
    }
    for (int e = tid; e < nb * nb; e += nth) X[(e / nb) * m + k0 + (e % nb)] = 0.0;
    __syncthreads();
    {  // A[:, j] = [0 on pivot rows; A] + Panel X (columns outside the panel), DMMA 8 x 8 tiles
      const int nt8 = (m + 7) / 8, pt = k0 / 8;
      const int lr = lane >> 2, lc = lane & 3;
      for (int it = wid; it < nt8 * nt8; it += nw) {
        const int tr = it / nt8, tc = it - tr * nt8;
        if (tc == pt) continue;
        const int R = tr * 8 + lr;
        const bool rok = R < m, rpiv = R >= k0 && R < k1;
        double cc[2];
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int J = tc * 8 + 2 * lc + e;
          cc[e] = (rok && !rpiv && J < m) ? A[R * m + J] : 0.0;
        }
        const int Jb = tc * 8 + lr;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int t = 4 * h + lc;
          const double a = (rok && t < nb) ? A[R * m + k0 + t] : 0.0;
          const double bb = (t < nb && Jb < m) ? X[t * m + Jb] : 0.0;
          dmma_ns(cc[0], cc[1], a, bb);
        }
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int J = tc * 8 + 2 * lc + e;
          if (rok && J < m) A[R * m + J] = cc[e];
        }
      }
    }
    __syncthreads();
  }
  if (tid == 0) {
    for (int c = 0; c < m; ++c) idx[c] = c;
    for (int c = m - 1; c >= 0; --c) {
      const int p = piv[c], t = idx[c];
      idx[c] = idx[p];
      idx[p] = t;
    }
  }
  __syncthreads();
  return s_info;
}

// ---- look-ahead form of gj_invert_smem_wp (same pivots, same operations per entry)
// Panel k's update is split: first the next panel's tile column (all warps), then
// warp 0 factors panel k + 1 in registers WHILE the other warps apply panel k to the
// remaining tile columns -- the panel's serial shuffle chain overlaps the bulk DMMA
// update instead of every other warp waiting for it at a barrier.  Two barriers per
// panel plus one between the phases.

// Warp 0: Gauss-Jordan on the panel columns [k0, k0 + nb) (registers, lane l holds
// rows l, l + 32, ...), pivots into piv, the factored panel written back to A.
template <int RPL>
__device__ __forceinline__ void gj_wp_panel(double *A, int m, int k0, int nb, double tol, int *piv, int *s_info,
                                            int lane) {
  double P[RPL][GJB];
#pragma unroll
  for (int s = 0; s < RPL; ++s) {
    const int r = lane + 32 * s;
#pragma unroll
    for (int t = 0; t < GJB; ++t) P[s][t] = (r < m && t < nb) ? A[r * m + k0 + t] : 0.0;
  }
  int info = 0;
#pragma unroll
  for (int tc = 0; tc < GJB; ++tc) {
    if (tc >= nb) break;
    const int c = k0 + tc;
    double bv = -1.0;
    int bi = m;
#pragma unroll
    for (int s = 0; s < RPL; ++s) {
      const int r = lane + 32 * s;
      const double v = fabs(P[s][tc]);
      if (r >= c && r < m && v > bv) {
        bv = v;
        bi = r;
      }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ov > bv || (ov == bv && oi < bi)) {
        bv = ov;
        bi = oi;
      }
    }
    if (!(bv >= tol) && info == 0) info = c + 1;
    const int sp = bi >> 5, lp = bi & 31, sc = c >> 5, lc = c & 31;
    double prow[GJB], crow[GJB];
#pragma unroll
    for (int t = 0; t < GJB; ++t) {
      double vp = 0.0, vc = 0.0;
#pragma unroll
      for (int s = 0; s < RPL; ++s) {
        vp = (s == sp) ? P[s][t] : vp;
        vc = (s == sc) ? P[s][t] : vc;
      }
      prow[t] = __shfl_sync(0xffffffffu, vp, lp);
      crow[t] = __shfl_sync(0xffffffffu, vc, lc);
    }
    const double pv = prow[tc];
    const double pinv = pv != 0.0 ? 1.0 / pv : 0.0;
    double newc[GJB];
#pragma unroll
    for (int t = 0; t < GJB; ++t) newc[t] = (t == tc) ? pinv : prow[t] * pinv;
#pragma unroll
    for (int s = 0; s < RPL; ++s) {
      const int r = lane + 32 * s;
      if (r == bi && bi != c) {
#pragma unroll
        for (int t = 0; t < GJB; ++t) P[s][t] = crow[t];
      }
      if (r == c) {
#pragma unroll
        for (int t = 0; t < GJB; ++t) P[s][t] = newc[t];
      } else {
        const double fr = P[s][tc];
#pragma unroll
        for (int t = 0; t < GJB; ++t)
          if (t != tc) P[s][t] = fma(-fr, newc[t], P[s][t]);
        P[s][tc] = -fr * pinv;
      }
    }
    if (lane == 0) piv[c] = bi;
  }
#pragma unroll
  for (int s = 0; s < RPL; ++s) {
    const int r = lane + 32 * s;
    if (r < m)
#pragma unroll
      for (int t = 0; t < GJB; ++t)
        if (t < nb) A[r * m + k0 + t] = P[s][t];
  }
  if (lane == 0 && info && *s_info == 0) *s_info = info;
}

// DMMA rank-nb update A[:, j] = [0 on pivot rows; A] + Panel X over the 8 x 8 tiles of
// the selected tile columns: mode 0 every column but the panel's (pt), 1 only pt + 1,
// 2 every column but pt and pt + 1.  Warps wslot, wslot + nws, ... walk the tiles.
__device__ __forceinline__ void gj_tile_update(double *A, const double *X, int m, int k0, int nb, int mode,
                                               int wslot, int nws, int lane) {
  const int k1 = k0 + nb, nt8 = (m + 7) / 8, pt = k0 / 8;
  const int nsel = mode == 0 ? nt8 - 1 : (mode == 1 ? 1 : nt8 - 2);
  const int lr = lane >> 2, lc = lane & 3;
  int tr = wslot, tci = 0;
  for (;;) {
    while (tr >= nt8) {
      tr -= nt8;
      ++tci;
    }
    if (tci >= nsel) break;
    const int tc = mode == 1 ? pt + 1 : (tci < pt ? tci : tci + (mode == 0 ? 1 : 2));
    const int R = tr * 8 + lr;
    const bool rok = R < m, rpiv = R >= k0 && R < k1;
    double cc[2];
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int J = tc * 8 + 2 * lc + e;
      cc[e] = (rok && !rpiv && J < m) ? A[R * m + J] : 0.0;
    }
    const int Jb = tc * 8 + lr;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int t = 4 * h + lc;
      const double a = (rok && t < nb) ? A[R * m + k0 + t] : 0.0;
      const double bb = (t < nb && Jb < m) ? X[t * m + Jb] : 0.0;
      dmma_ns(cc[0], cc[1], a, bb);
    }
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int J = tc * 8 + 2 * lc + e;
      if (rok && J < m) A[R * m + J] = cc[e];
    }
    tr += nws;
  }
}

template <int RPL>
__device__ int gj_invert_smem_la(double *A, int m, double tol, double *X, int *piv, int *idx) {
  __shared__ int s_info;
  const int tid = threadIdx.x, nth = blockDim.x, lane = tid & 31, wid = tid >> 5, nw = nth >> 5;
  if (tid == 0) s_info = 0;
  __syncthreads();
  if (wid == 0) gj_wp_panel<RPL>(A, m, 0, min(GJB, m), tol, piv, &s_info, lane);
  __syncthreads();
  for (int k0 = 0; k0 < m; k0 += GJB) {
    const int nb = min(GJB, m - k0), k1 = k0 + nb;
    // the panel's row interchanges on the other columns (pivot order), X = pivot rows
    for (int j = tid; j < m; j += nth) {
      if (j >= k0 && j < k1) continue;
      for (int c = k0; c < k1; ++c) {
        const int p = piv[c];
        if (p != c) {
          const double t1 = A[c * m + j];
          A[c * m + j] = A[p * m + j];
          A[p * m + j] = t1;
        }
      }
      for (int t = 0; t < nb; ++t) X[t * m + j] = A[(k0 + t) * m + j];
    }
    for (int e = tid; e < nb * nb; e += nth) X[(e / nb) * m + k0 + (e % nb)] = 0.0;
    __syncthreads();
    if (k1 < m) {
      gj_tile_update(A, X, m, k0, nb, 1, wid, nw, lane);  // the next panel's columns first
      __syncthreads();
      if (wid == 0)
        gj_wp_panel<RPL>(A, m, k1, min(GJB, m - k1), tol, piv, &s_info, lane);
      else
        gj_tile_update(A, X, m, k0, nb, 2, wid - 1, nw - 1, lane);
    } else {
      gj_tile_update(A, X, m, k0, nb, 0, wid, nw, lane);
    }
    __syncthreads();
  }
  if (tid == 0) {
    for (int c = 0; c < m; ++c) idx[c] = c;
    for (int c = m - 1; c >= 0; --c) {
      const int p = piv[c], t = idx[c];
      idx[c] = idx[p];
      idx[p] = t;
    }
  }
  __syncthreads();
  return s_info;
}

// ---- look-ahead form without row interchanges (gj_invert_smem_lr)
// The pivot rows stay where they are: column c eliminates with the unused row of
// largest |a| (lowest row on ties -- on exact ties a different, equally valid pivot
// than dgetrf's position order; the inverse agrees to rounding), recorded in
// prow_of[c]; X copies the panel's pivot rows, the update zeroes them, and the row
// order of the result is restored once at the end by replaying the equivalent
// interchanges (the inverse of P A, then the column permutation as before).  No
// interchange pass over the matrix per panel, no displaced-row shuffles in the panel.
// reciprocal: rcp.approx + a cubic and a Newton step (correct to the last bit or two; 0 -> 0)
__device__ __forceinline__ double rt_rcp(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double e = fma(-x, r, 1.0);
  e = fma(e, e, e);  // r (1 + e + e^2): cubic step
  r = fma(r, e, r);
  e = fma(-x, r, 1.0);
  r = fma(r, e, r);
  return x != 0.0 ? r : 0.0;
}

template <int RPL>
__device__ __forceinline__ void gj_lr_panel(double *A, int m, int k0, int nb, double tol, int *prow_of,
                                            int8_t *used_in, int *s_info, double *bc, int lane) {
  // the pivot search and broadcast of rt_panel (redux.sync over a high-word key, speculative
  // reciprocals, pivot row through shared memory bc[9]; ties and near-ties to the lowest row)
  double P[RPL][8];
  unsigned elig = 0;
#pragma unroll
  for (int s = 0; s < RPL; ++s) {
    const int r = lane + 32 * s;
    if (r < m && used_in[r] < 0) elig |= 1u << s;
#pragma unroll
    for (int t = 0; t < GJB; ++t) P[s][t] = (r < m && t < nb) ? A[r * m + k0 + t] : 0.0;
  }
  int info = 0;
  const int pt = k0 / GJB;
#pragma unroll
  for (int tc = 0; tc < GJB; ++tc) {
    if (tc >= nb) break;
    const int c = k0 + tc;
    unsigned key = 0;
    double rc[RPL];
#pragma unroll
    for (int s = 0; s < RPL; ++s) {
      const double v = P[s][tc];
      rc[s] = rt_rcp(v);
      const unsigned k = ((elig >> s) & 1u)
                             ? (((unsigned)__double2hiint(v) & 0x7FFFFF00u) | (unsigned)(255 - (lane + 32 * s)))
                             : 0u;
      key = max(key, k);
    }
    const unsigned gk = __reduce_max_sync(0xffffffffu, key);
    const int bi = 255 - (int)(gk & 255u), lp = bi & 31, sp = bi >> 5;
    const bool isl = lane == lp;
    if (isl) {
#pragma unroll
      for (int s = 0; s < RPL; ++s)
        if (s == sp) {
#pragma unroll
          for (int t = 0; t < GJB; ++t) bc[t] = P[s][t];
          bc[8] = rc[s];
        }
    }
    __syncwarp();
    double prow_v[GJB];
#pragma unroll
    for (int t = 0; t < GJB; ++t) prow_v[t] = bc[t];
    const double pinv = bc[8];
    __syncwarp();
    if (!(fabs(prow_v[tc]) >= tol) && info == 0) info = c + 1;
#pragma unroll
    for (int s = 0; s < RPL; ++s) {
      const double frp = P[s][tc] * pinv;
#pragma unroll
      for (int t = 0; t < GJB; ++t)
        if (t != tc) P[s][t] = fma(-frp, prow_v[t], P[s][t]);
      P[s][tc] = -frp;
    }
    double keep[GJB];
#pragma unroll
    for (int t = 0; t < GJB; ++t) keep[t] = (t == tc) ? pinv : prow_v[t] * pinv;
#pragma unroll
    for (int s = 0; s < RPL; ++s)
      if (s == sp) {
#pragma unroll
        for (int t = 0; t < GJB; ++t) P[s][t] = isl ? keep[t] : P[s][t];
      }
    if (isl) elig &= ~(1u << sp);
    if (lane == 0) {
      prow_of[c] = bi;
      used_in[bi] = (int8_t)(pt & 127);
    }
  }
#pragma unroll
  for (int s = 0; s < RPL; ++s) {
    const int r = lane + 32 * s;
    if (r < m)
#pragma unroll
      for (int t = 0; t < GJB; ++t)
        if (t < nb) A[r * m + k0 + t] = P[s][t];
  }
  if (lane == 0 && info && *s_info == 0) *s_info = info;
}

// gj_tile_update with the panel's pivot rows marked in used_in (== pt & 127).
__device__ __forceinline__ void gj_lr_tile_update(double *A, const double *X, const int8_t *used_in, int m, int k0,
                                                  int nb, int mode, int wslot, int nws, int lane) {
  const int nt8 = (m + 7) / 8, pt = k0 / 8;
  const int nsel = mode == 0 ? nt8 - 1 : (mode == 1 ? 1 : nt8 - 2);
  const int lr = lane >> 2, lc = lane & 3;
  const int8_t mark = (int8_t)(pt & 127);
  int tr = wslot, tci = 0;
  for (;;) {
    while (tr >= nt8) {
      tr -= nt8;
      ++tci;
    }
    if (tci >= nsel) break;
    const int tc = mode == 1 ? pt + 1 : (tci < pt ? tci : tci + (mode == 0 ? 1 : 2));
    const int R = tr * 8 + lr;
    const bool rok = R < m, rpiv = rok && used_in[R] == mark;
    double cc[2];
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int J = tc * 8 + 2 * lc + e;
      cc[e] = (rok && !rpiv && J < m) ? A[R * m + J] : 0.0;
    }
    const int Jb = tc * 8 + lr;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int t = 4 * h + lc;
      const double a = (rok && t < nb) ? A[R * m + k0 + t] : 0.0;
      const double bb = (t < nb && Jb < m) ? X[t * m + Jb] : 0.0;
      dmma_ns(cc[0], cc[1], a, bb);
    }
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int J = tc * 8 + 2 * lc + e;
      if (rok && J < m) A[R * m + J] = cc[e];
    }
    tr += nws;
  }
}

// Column-strip form of gj_lr_tile_update (round 2): a warp takes whole tile columns J
// (mode 1, the single look-ahead column: its row tiles split across the warps), so the
// B fragments (the pivot rows, kept in fragment order XF[J][h][lane]) are loaded once per
// column; C moves as one 16-byte access per lane (m even: conflict-free, row stride m / 2
// 16-byte words); the rows that pivoted in this panel are masked by the per-lane-row bit
// masks pm[lr] (bit I: row 8 I + lr).  Reads past row m stay inside the buffer (A is
// followed by >= 8 m doubles of X) and are discarded; only stores are predicated.
template <bool EVEN>
__device__ __forceinline__ void gj_lr_strip_update(double *A, const double *XF, const unsigned *pm, int m, int k0,
                                                   int nb, int mode, int wslot, int nws, int lane) {
  const int nt8 = (m + 7) / 8, pt = k0 / 8;
  const int ncol = mode == 0 ? nt8 - 1 : (mode == 1 ? 1 : nt8 - 2);
  const int lr = lane >> 2, lc = lane & 3;
  const unsigned pmk = pm[lr];
  const bool ua0 = lc < nb, ua1 = 4 + lc < nb;
  const int cstep = mode == 1 ? 1 : nws, istep = mode == 1 ? nws : 1;
  for (int ci = mode == 1 ? 0 : wslot; ci < ncol; ci += cstep) {
    const int J = mode == 1 ? pt + 1 : (ci < pt ? ci : ci + (mode == 0 ? 1 : 2));
    const double b0 = XF[(J * 2) * 32 + lane], b1 = XF[(J * 2 + 1) * 32 + lane];
    const int C0 = J * 8 + 2 * lc;
    const bool cok = C0 < m, cok1 = C0 + 1 < m;
    const double *ap = A + lr * m + k0 + lc;
    double *cp = A + lr * m + C0;
#pragma unroll 3
    for (int I = mode == 1 ? wslot : 0; I < nt8; I += istep) {
      const int off = I * 8 * m;
      double a0 = ap[off], a1 = ap[off + 4];
      a0 = ua0 ? a0 : 0.0;
      a1 = ua1 ? a1 : 0.0;
      double c0, c1;
      if (EVEN) {
        const double2 v = *reinterpret_cast<const double2 *>(cp + off);
        c0 = v.x;
        c1 = v.y;
      } else {
        c0 = cp[off];
        c1 = cp[off + 1];
      }
      const bool z = (pmk >> I) & 1u;
      c0 = z ? 0.0 : c0;
      c1 = z ? 0.0 : c1;
      dmma_ns(c0, c1, a0, b0);
      dmma_ns(c0, c1, a1, b1);
      if (I * 8 + lr < m) {
        if (EVEN) {
          if (cok) *reinterpret_cast<double2 *>(cp + off) = make_double2(c0, c1);
        } else {
          if (cok) cp[off] = c0;
          if (cok1) cp[off + 1] = c1;
        }
      }
    }
  }
}

// On return rowmap[c] = the physical row of A holding row c of (P A)^{-1} and idx the
// column permutation as in gj_invert_smem: D^{-1}[rho][sig] = A[rowmap[rho]][idx[sig]].
// Shared scratch: piv, idx, rowmap, tmp (m ints each), used_in (m bytes).
template <int RPL>
__device__ int gj_invert_smem_lr(double *A, int m, double tol, double *X, int *piv, int *idx, int8_t *used_in,
                                 int *rowmap, int *tmp) {
  __shared__ int s_info;
  const int tid = threadIdx.x, nth = blockDim.x, lane = tid & 31, wid = tid >> 5, nw = nth >> 5;
  if (tid == 0) s_info = 0;
  for (int r = tid; r < m; r += nth) used_in[r] = -1;
  __syncthreads();
  int *prow_of = rowmap;  // the pivot row of every column during the elimination
  __shared__ double s_bc[16];
  if (wid == 0) gj_lr_panel<RPL>(A, m, 0, min(GJB, m), tol, prow_of, used_in, &s_info, s_bc, lane);
  __syncthreads();
  __shared__ unsigned s_pm[8];
  const bool even = (m & 1) == 0;
  const int nt8 = (m + 7) / 8;
  for (int k0 = 0; k0 < m; k0 += GJB) {
    const int nb = min(GJB, m - k0), k1 = k0 + nb;
    // XF = the panel's pivot rows (other columns) in B-fragment order [J][h][lane]
    for (int e = tid; e < nt8 * 64; e += nth) {
      const int J = e >> 6, h = (e >> 5) & 1, ln = e & 31, t = 4 * h + (ln & 3), j = J * 8 + (ln >> 2);
      const bool inp = j >= k0 && j < k1;
      X[e] = (t < nb && j < m && !inp) ? A[prow_of[k0 + t] * m + j] : 0.0;
    }
    if (tid < 8) {
      unsigned mk = 0;
      for (int t = 0; t < nb; ++t) {
        const int r = prow_of[k0 + t];
        if ((r & 7) == tid) mk |= 1u << (r >> 3);
      }
      s_pm[tid] = mk;
    }
    __syncthreads();
    if (k1 < m) {
      if (even) gj_lr_strip_update<true>(A, X, s_pm, m, k0, nb, 1, wid, nw, lane);
      else gj_lr_strip_update<false>(A, X, s_pm, m, k0, nb, 1, wid, nw, lane);
      __syncthreads();
      if (wid == 0)
        gj_lr_panel<RPL>(A, m, k1, min(GJB, m - k1), tol, prow_of, used_in, &s_info, s_bc, lane);
      else if (even)
        gj_lr_strip_update<true>(A, X, s_pm, m, k0, nb, 2, wid - 1, nw - 1, lane);
      else
        gj_lr_strip_update<false>(A, X, s_pm, m, k0, nb, 2, wid - 1, nw - 1, lane);
    } else {
      if (even) gj_lr_strip_update<true>(A, X, s_pm, m, k0, nb, 0, wid, nw, lane);
      else gj_lr_strip_update<false>(A, X, s_pm, m, k0, nb, 0, wid, nw, lane);
    }
    __syncthreads();
  }
  if (tid == 0) {
    // replay the equivalent interchanges: position c receives row prow_of[c]
    int *pos2row = tmp, *row2pos = piv;
    for (int c = 0; c < m; ++c) pos2row[c] = row2pos[c] = c;
    for (int c = 0; c < m; ++c) {
      const int pr = rowmap[c], pp = row2pos[pr], rc = pos2row[c];
      pos2row[c] = pr;
      pos2row[pp] = rc;
      row2pos[pr] = c;
      row2pos[rc] = pp;
      rowmap[c] = pp;  // the dgetrf-style pivot position of column c
    }
    for (int c = 0; c < m; ++c) idx[c] = c;
    for (int c = m - 1; c >= 0; --c) {
      const int p = rowmap[c], t = idx[c];
      idx[c] = idx[p];
      idx[p] = t;
    }
    for (int c = 0; c < m; ++c) rowmap[c] = pos2row[c];
  }
  __syncthreads();
  return s_info;
}

// Warp-per-block Gauss-Jordan (m <= 32 RPL): the same elimination as
// gj_invert_smem_wp (identical pivots and operations per entry) carried out by one
// warp on its own block -- panel in registers, interchanges and DMMA rank-GJB
// updates by the same warp -- so blocks never wait at CTA barriers and a CTA keeps
// several blocks in flight (one per warp).
template <int RPL>
__device__ int gj_invert_warp(double *A, int m, double tol, double *X, int *piv, int *idx, int lane) {
  int info = 0;
  for (int k0 = 0; k0 < m; k0 += GJB) {
    const int nb = min(GJB, m - k0), k1 = k0 + nb;
    double P[RPL][GJB];
#pragma unroll
    for (int s = 0; s < RPL; ++s) {
      const int r = lane + 32 * s;
#pragma unroll
      for (int t = 0; t < GJB; ++t) P[s][t] = (r < m && t < nb) ? A[r * m + k0 + t] : 0.0;
    }
#pragma unroll
    for (int tc = 0; tc < GJB; ++tc) {
      if (tc >= nb) break;
      const int c = k0 + tc;
      double bv = -1.0;
      int bi = m;
#pragma unroll
      for (int s = 0; s < RPL; ++s) {
        const int r = lane + 32 * s;
        const double v = fabs(P[s][tc]);
        if (r >= c && r < m && v > bv) {
          bv = v;
          bi = r;
        }
      }
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ov > bv || (ov == bv && oi < bi)) {
          bv = ov;
          bi = oi;
        }
      }
      if (!(bv >= tol) && info == 0) info = c + 1;
      const int sp = bi >> 5, lp = bi & 31, sc = c >> 5, lc = c & 31;
      double prow[GJB], crow[GJB];
#pragma unroll
      for (int t = 0; t < GJB; ++t) {
        double vp = 0.0, vc = 0.0;
#pragma unroll
        for (int s = 0; s < RPL; ++s) {
          vp = (s == sp) ? P[s][t] : vp;
          vc = (s == sc) ? P[s][t] : vc;
        }
        prow[t] = __shfl_sync(0xffffffffu, vp, lp);
        crow[t] = __shfl_sync(0xffffffffu, vc, lc);
      }
      const double pv = prow[tc];
      const double pinv = pv != 0.0 ? 1.0 / pv : 0.0;
      double newc[GJB];
#pragma unroll
      for (int t = 0; t < GJB; ++t) newc[t] = (t == tc) ? pinv : prow[t] * pinv;
#pragma unroll
      for (int s = 0; s < RPL; ++s) {
        const int r = lane + 32 * s;
        if (r == bi && bi != c) {
#pragma unroll
          for (int t = 0; t < GJB; ++t) P[s][t] = crow[t];
        }
        if (r == c) {
#pragma unroll
          for (int t = 0; t < GJB; ++t) P[s][t] = newc[t];
        } else {
          const double fr = P[s][tc];
#pragma unroll
          for (int t = 0; t < GJB; ++t)
            if (t != tc) P[s][t] = fma(-fr, newc[t], P[s][t]);
          P[s][tc] = -fr * pinv;
        }
      }
      if (lane == 0) piv[c] = bi;
    }
#pragma unroll
    for (int s = 0; s < RPL; ++s) {
      const int r = lane + 32 * s;
      if (r < m)
#pragma unroll
        for (int t = 0; t < GJB; ++t)
          if (t < nb) A[r * m + k0 + t] = P[s][t];
    }
    __syncwarp();
    for (int j = lane; j < m; j += 32) {
      if (j >= k0 && j < k1) continue;
      for (int c = k0; c < k1; ++c) {
        const int p = piv[c];
        if (p != c) {
          const double t1 = A[c * m + j];
          A[c * m + j] = A[p * m + j];
          A[p * m + j] = t1;
        }
      }
      for (int t = 0; t < nb; ++t) X[t * m + j] = A[(k0 + t) * m + j];
    }
    for (int e = lane; e < nb * nb; e += 32) X[(e / nb) * m + k0 + (e % nb)] = 0.0;
    __syncwarp();
    {
      const int nt8 = (m + 7) / 8, pt = k0 / 8;
      const int lr = lane >> 2, lcc = lane & 3;
      for (int it = 0; it < nt8 * nt8; ++it) {
        const int tr = it / nt8, tcl = it - tr * nt8;
        if (tcl == pt) continue;
        const int R = tr * 8 + lr;
        const bool rok = R < m, rpiv = R >= k0 && R < k1;
        double cc[2];
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int J = tcl * 8 + 2 * lcc + e;
          cc[e] = (rok && !rpiv && J < m) ? A[R * m + J] : 0.0;
        }
        const int Jb = tcl * 8 + lr;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int t = 4 * h + lcc;
          const double a = (rok && t < nb) ? A[R * m + k0 + t] : 0.0;
          const double bb = (t < nb && Jb < m) ? X[t * m + Jb] : 0.0;
          dmma_ns(cc[0], cc[1], a, bb);
        }
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int J = tcl * 8 + 2 * lcc + e;
          if (rok && J < m) A[R * m + J] = cc[e];
        }
      }
    }
    __syncwarp();
  }
  if (lane == 0) {
    for (int c = 0; c < m; ++c) idx[c] = c;
    for (int c = m - 1; c >= 0; --c) {
      const int p = piv[c], t = idx[c];
      idx[c] = idx[p];
      idx[p] = t;
    }
  }
  __syncwarp();
  return info;
}

// One warp per (patch, slab) block, WPB blocks per CTA (shared memory: WPB private
// m x m matrices), blocks b = blockIdx.x WPB + w over npatch N: assembly as in
// k_ns_factor, warp-per-block Gauss-Jordan, column-major inverse out.
template <int NQ, int WPB, int RPL>
__global__ void __launch_bounds__(32 * WPB) k_ns_factor_warp(int mp, int N, int64_t nblk, int64_t mstride,
                                                             const int32_t *__restrict__ pnodes,
                                                             const double *__restrict__ Mv,
                                                             const double *__restrict__ KGv,
                                                             const double *__restrict__ conv, NSTime tm,
                                                             double *__restrict__ out, int32_t *__restrict__ info,
                                                             const int32_t *__restrict__ ppos,
                                                             const int32_t *__restrict__ pvv) {
  extern __shared__ __align__(16) double smem[];
  const int m = NQ * mp;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const size_t per = ns_factor_warp_doubles(m, mp);
  double *A = smem + w * per, *X = A + (size_t)m * m;
  int *piv = (int *)(X + GJB * m);
  int *idx = piv + m;
  int *nodes = idx + m;
  const int64_t NT = (int64_t)N * NQ;
  for (int64_t blk = (int64_t)blockIdx.x * WPB + w; blk < nblk; blk += (int64_t)gridDim.x * WPB) {
    const int64_t p = blk / N;
    const int n = (int)(blk - p * N);
    for (int i = lane; i < mp; i += 32) nodes[i] = pnodes[p * mp + i];
    __syncwarp();
    const int npair = mp * mp;
    for (int e = lane; e < npair; e += 32) {
      const int ii = e / mp, jj = e - ii * mp;
      const bool pad = nodes[ii] < 0 || nodes[jj] < 0;
      const int64_t pe = (p * mp + ii) * mp + jj;
      const int pos = pad ? -1 : __ldg(ppos + pe);
      const int vv = pad ? -1 : __ldg(pvv + pe);
      const double mv = pos >= 0 ? __ldg(Mv + pos) : 0.0, kg = pos >= 0 ? __ldg(KGv + pos) : 0.0;
      double cv[NQ];
      const double *cp = conv + (int64_t)(vv >= 0 ? vv : 0) * NT + (int64_t)n * NQ;
#pragma unroll
      for (int c = 0; c < NQ; ++c) cv[c] = (pos >= 0 && vv >= 0) ? __ldg(cp + c) : 0.0;
#pragma unroll
      for (int a = 0; a < NQ; ++a)
#pragma unroll
        for (int bb = 0; bb < NQ; ++bb) {
          const int rho = ii * NQ + a, sig = jj * NQ + bb;
          double v;
          if (pad) {
            v = (rho == sig) ? 1.0 : 0.0;
          } else if (pos < 0) {
            v = 0.0;
          } else {
            v = tm.CE[a * NQ + bb] * mv + tm.Mt[a * NQ + bb] * kg;
            if (vv >= 0)
#pragma unroll
              for (int c = 0; c < NQ; ++c) v = fma(tm.T[(a * NQ + bb) * NQ + c], cv[c], v);
          }
          A[rho * m + sig] = v;
        }
    }
    __syncwarp();
    double rn = 0.0;  // max row norm (R10 tolerance)
    for (int r = lane; r < m; r += 32) {
      double sum = 0.0;
      for (int c = 0; c < m; ++c) sum += fabs(A[r * m + c]);
      rn = fmax(rn, sum);
    }
    for (int o = 16; o; o >>= 1) rn = fmax(rn, __shfl_xor_sync(0xffffffffu, rn, o));
    const int st = gj_invert_warp<RPL>(A, m, 1e-14 * rn, X, piv, idx, lane);
    double *o = out + blk * mstride;  // column-major: o[sig m + rho] = D^{-1}[rho][sig]
    for (int e = lane; e < m * m; e += 32) {
      const int sig = e / m, rho = e - sig * m;
      o[e] = A[rho * m + idx[sig]];
    }
    if (lane == 0) info[blk] = st;
    __syncwarp();
  }
}

// H4: D_{p,n} = R_p A_nn R_p^T (R9) assembled row-major (stride m) into shared A from the
// per-patch pair tables; pad DoFs (node < 0) get identity rows.  The caller syncs after.
template <int NQ>
__device__ __forceinline__ void ns_assemble_block(double *A, int *nodes, int mp, int64_t p, int n, int N,
                                                  const int32_t *__restrict__ pnodes, const double *__restrict__ Mv,
                                                  const double *__restrict__ KGv, const double *__restrict__ conv,
                                                  const NSTime &tm, const int32_t *__restrict__ ppos,
                                                  const int32_t *__restrict__ pvv) {
  const int m = NQ * mp, tid = threadIdx.x;
  const int64_t NT = (int64_t)N * NQ;
  for (int i = tid; i < mp; i += blockDim.x) nodes[i] = pnodes[p * mp + i];
  __syncthreads();
  // thread per node pair (i, j): the pair's CSR position, mass / stiffness values
  // and convection values are loaded once for its NQ x NQ entries (node-major:
  // rho = i NQ + a, sig = j NQ + bb); two pairs per iteration for more loads in flight
  const int npair = mp * mp;
  for (int e0 = tid; e0 < npair; e0 += 2 * blockDim.x) {
    int pos[2], vv[2], ii[2], jj[2];
    bool pad[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int e = e0 + h * blockDim.x;
      const bool ok = e < npair;
      ii[h] = ok ? e / mp : 0;
      jj[h] = ok ? e - ii[h] * mp : 0;
      pad[h] = !ok || nodes[ii[h]] < 0 || nodes[jj[h]] < 0;
      const int64_t pe = (p * mp + ii[h]) * mp + jj[h];
      pos[h] = (!pad[h]) ? __ldg(ppos + pe) : -1;
      vv[h] = (!pad[h]) ? __ldg(pvv + pe) : -1;
    }
    double mv[2], kg[2], cv[2][NQ];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      mv[h] = pos[h] >= 0 ? __ldg(Mv + pos[h]) : 0.0;
      kg[h] = pos[h] >= 0 ? __ldg(KGv + pos[h]) : 0.0;
      const double *cp = conv + (int64_t)(vv[h] >= 0 ? vv[h] : 0) * NT + (int64_t)n * NQ;
#pragma unroll
      for (int c = 0; c < NQ; ++c) cv[h][c] = (pos[h] >= 0 && vv[h] >= 0) ? __ldg(cp + c) : 0.0;
    }
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      if (e0 + h * blockDim.x >= npair) continue;
#pragma unroll
      for (int a = 0; a < NQ; ++a)
#pragma unroll
        for (int bb = 0; bb < NQ; ++bb) {
          const int rho = ii[h] * NQ + a, sig = jj[h] * NQ + bb;
          double v;
          if (pad[h]) {
            v = (rho == sig) ? 1.0 : 0.0;
          } else if (pos[h] < 0) {
            v = 0.0;
          } else {
            v = tm.CE[a * NQ + bb] * mv[h] + tm.Mt[a * NQ + bb] * kg[h];
            if (vv[h] >= 0)
#pragma unroll
              for (int c = 0; c < NQ; ++c) v = fma(tm.T[(a * NQ + bb) * NQ + c], cv[h][c], v);
          }
          A[rho * m + sig] = v;
        }
    }
  }
}

// One CTA per (patch p = blockIdx.x, slab n = blockIdx.y): assemble D_{p,n} (pad
// DoFs: identity rows), invert, write the row-major inverse to
// out[(p N + n) mstride ...].  info[p N + n] = 0 or 1 + singular column.
template <int NQ, int NTH, int RPL, int LA = 0>  // LA: 0 gj_invert_smem_wp, 1 _la, 2 _lr
__global__ void __launch_bounds__(NTH, (LA && NTH == 128) ? 4 : 1) k_ns_factor(int mp, int N, int64_t mstride, const int32_t *__restrict__ pnodes,
                                                   const int32_t *__restrict__ rowptr, const int32_t *__restrict__ col,
                                                   const double *__restrict__ Mv, const double *__restrict__ KGv,
                                                   int64_t nvrow, const int32_t *__restrict__ vvptr,
                                                   const double *__restrict__ conv, NSTime tm,
                                                   double *__restrict__ out, int32_t *__restrict__ info,
                                                   const int32_t *__restrict__ ppos, const int32_t *__restrict__ pvv,
                                                   int n0, int nwin) {
  extern __shared__ __align__(16) double smem[];
  const int m = NQ * mp;
  double *A = smem, *X = smem + (int64_t)m * m;  // X: ns_factor_xdoubles(m)
  int *piv = (int *)(X + ns_factor_xdoubles(m));
  int *idx = piv + m;
  int *nodes = idx + m;
  int *rowmap = nodes + mp, *tmp = rowmap + m;  // LA == 2 only (ns_factor_smem_lr)
  int8_t *used_in = (int8_t *)(tmp + m);
  __shared__ double s_red[32];
  const int64_t p = blockIdx.x;
  const int n = n0 + blockIdx.y;  // slab window [n0, n0 + nwin)
  const int64_t NT = (int64_t)N * NQ;
  const int tid = threadIdx.x;
  ns_assemble_block<NQ>(A, nodes, mp, p, n, N, pnodes, Mv, KGv, conv, tm, ppos, pvv);
  __syncthreads();
  double rn = 0.0;  // max row norm (R10 tolerance)
  for (int r = tid; r < m; r += blockDim.x) {
    double s = 0.0;
    for (int c = 0; c < m; ++c) s += fabs(A[r * m + c]);
    rn = fmax(rn, s);
  }
  for (int o = 16; o; o >>= 1) rn = fmax(rn, __shfl_xor_sync(0xffffffffu, rn, o));
  if ((tid & 31) == 0) s_red[tid >> 5] = rn;
  __syncthreads();
  double mx = 0.0;
  for (int w = 0; w < (int)(blockDim.x >> 5); ++w) mx = fmax(mx, s_red[w]);
  static_assert(GJB == 8, "panel width");
  int st;
  if constexpr (RPL > 0 && LA == 2) st = gj_invert_smem_lr<RPL>(A, m, 1e-14 * mx, X, piv, idx, used_in, rowmap, tmp);
  else if constexpr (RPL > 0 && LA == 1) st = gj_invert_smem_la<RPL>(A, m, 1e-14 * mx, X, piv, idx);  // m <= 32 RPL
  else if constexpr (RPL > 0) st = gj_invert_smem_wp<RPL>(A, m, 1e-14 * mx, X, piv, idx);
  else st = gj_invert_smem(A, m, 1e-14 * mx, X, piv, idx);
  double *o = out + (p * nwin + blockIdx.y) * mstride;  // column-major: o[sig m + rho] = D^{-1}[rho][sig]
  for (int e = tid; e < m * m; e += blockDim.x) {
    const int sig = e / m, rho = e - sig * m;
    o[e] = A[(LA == 2 ? rowmap[rho] : rho) * m + idx[sig]];
  }
  if (tid == 0) info[p * N + n] = st;
}

// ---- H5 register-tiled Gauss-Jordan (k_ns_factor_rt, m <= 96; round 2)
// The block lives in DMMA accumulator fragments for the whole elimination: tile
// column J (8 columns, M = 8 NT padded; pad rows / columns = identity) belongs to
// accumulator warp J mod W, two tile columns per warp, so the rank-8 update of every
// panel reads only the factored panel (A fragments) and the pivot rows (B fragments)
// from shared memory -- the m^2 matrix itself is never re-read or re-written (the
// shared-memory kernel moves the whole matrix through shared memory once per panel:
// 83 % L1 busy, 56-66 % bank conflicts, ncu round 2).  A dedicated panel warp
// factors panel K+1 (columns in registers, no row interchanges as in
// gj_invert_smem_lr) while the accumulator warps apply panel K: the owner of tile
// column K+1 updates it first, hands it over through shared memory (named barrier
// 1), and the panel warp's pivot search is one redux.sync over a 32-bit key
// (|a| rounded to 16 mantissa bits, ties and near-ties to the lowest row -- a
// partial pivot within 2^-16 of the column maximum, R10) overlapped with each
// lane's speculative reciprocal of its own best candidate.  The result rows are the
// pivot rows of the unpermuted elimination: D^{-1}[rho][sig] = A[prow[rho]][q[sig]]
// with q the inverse of prow (DESIGN R10).
constexpr int RT_PS = 9;  // row stride of the panel hand-over buffer (odd: conflict-free row reads)


// Panel K (columns k0 .. k0+nb) from Pin (M x RT_PS, current values) -> Pf (A-fragment
// order [I][h][lane]) and the pivot records prow / used / tpos; one warp.  Row r is
// slot s = r / 32 of lane r % 32; the pivot is chosen by one redux.sync, every lane's
// reciprocals computed speculatively while it is in flight, and the pivot row and its
// reciprocal reach all lanes through shared memory (bc: 9 doubles; tools/panel_bench.cu:
// 378 cycles per column standalone against 442 with shuffles and an F2F key).
template <int M>
__device__ __forceinline__ void rt_panel(const double *Pin, double *Pf, int m, int K, int nb, double tol, int *prow,
                                         int8_t *used, int8_t *tpos, int *s_info, unsigned *pmask, double *bc,
                                         int lane) {
  constexpr int RPL = (M + 31) / 32;
  const int k0 = 8 * K;
  double P[RPL][8];
  unsigned elig = 0;
#pragma unroll
  for (int s = 0; s < RPL; ++s) {
    const int r = lane + 32 * s;
    if (r < m && used[r] < 0) elig |= 1u << s;
#pragma unroll
    for (int t = 0; t < 8; ++t) P[s][t] = (r < M) ? Pin[r * RT_PS + t] : 0.0;
  }
  int mybi = 0, sing = 0;
#pragma unroll
  for (int tc = 0; tc < 8; ++tc) {
    if (tc >= nb) break;
    // key = high word of |a| (13 mantissa bits) | (255 - row); every lane's reciprocals speculatively
    unsigned key = 0;
    double rc[RPL];
#pragma unroll
    for (int s = 0; s < RPL; ++s) {
      const double v = P[s][tc];
      rc[s] = rt_rcp(v);
      const unsigned k = ((elig >> s) & 1u)
                             ? (((unsigned)__double2hiint(v) & 0x7FFFFF80u) | (unsigned)(255 - (lane + 32 * s)))
                             : 0u;
      key = max(key, k);
    }
    const unsigned gk = __reduce_max_sync(0xffffffffu, key);
    const int bi = 255 - (int)(gk & 255u), lp = bi & 31, sp = bi >> 5;
    const bool isl = lane == lp;
    // the pivot row and its reciprocal through shared memory (one store set, broadcast loads)
    if (isl) {
#pragma unroll
      for (int s = 0; s < RPL; ++s)
        if (s == sp) {
#pragma unroll
          for (int t = 0; t < 8; ++t) bc[t] = P[s][t];
          bc[8] = rc[s];
        }
    }
    __syncwarp();
    double prow_v[8];
#pragma unroll
    for (int t = 0; t < 8; ++t) prow_v[t] = bc[t];
    const double pinv = bc[8];
    __syncwarp();
    const double pv = prow_v[tc];
#pragma unroll
    for (int s = 0; s < RPL; ++s) {  // rows -= (a_r,c / pivot) x pivot row
      const double frp = P[s][tc] * pinv;
#pragma unroll
      for (int t = 0; t < 8; ++t)
        if (t != tc) P[s][t] = fma(-frp, prow_v[t], P[s][t]);
      P[s][tc] = -frp;
    }
    double keep[8];  // the pivot row: scaled by 1 / pivot, its column entry = 1 / pivot
#pragma unroll
    for (int t = 0; t < 8; ++t) keep[t] = (t == tc) ? pinv : prow_v[t] * pinv;
#pragma unroll
    for (int s = 0; s < RPL; ++s)
      if (s == sp) {  // warp-uniform
#pragma unroll
        for (int t = 0; t < 8; ++t) P[s][t] = isl ? keep[t] : P[s][t];
      }
    if (isl) elig &= ~(1u << sp);
    if (lane == tc) mybi = bi;
    if (!(fabs(pv) >= tol) && sing == 0) sing = k0 + tc + 1;
  }
#pragma unroll
  for (int s = 0; s < RPL; ++s) {
    const int r = lane + 32 * s;
    if (r < M)
#pragma unroll
      for (int t = 0; t < 8; ++t)
        Pf[((r >> 3) * 2 + (t >> 2)) * 32 + (((r & 7) << 2) | (t & 3))] = (t < nb) ? P[s][t] : 0.0;
  }
  // the pivot rows of this panel as per-lane-row masks: bit I of pmask[lr] = row 8 I + lr pivoted
  unsigned pmk = 0;
#pragma unroll
  for (int t = 0; t < 8; ++t) {
    const int bt = __shfl_sync(0xffffffffu, mybi, t);
    if (t < nb && (bt & 7) == lane) pmk |= 1u << (bt >> 3);
  }
  if (lane < 8) pmask[(K & 1) * 8 + lane] = pmk;
  if (lane < nb) {
    prow[k0 + lane] = mybi;
    used[mybi] = (int8_t)K;
    tpos[mybi] = (int8_t)lane;
  }
  if (lane == 0 && sing && *s_info == 0) *s_info = sing;
}

// Rank-8 update of one (TWO = false) or two owned tile columns with panel K: acc += Pf X
// (the pivot rows of panel K were reset to zero when their X rows were written).
template <int NT, bool TWO>
__device__ __forceinline__ void rt_update(double (&acc0)[NT][2], double (&acc1)[NT][2], const double *Pf,
                                          const double *X, int J0, int J1, unsigned pm, int lane) {
  const double b00 = X[(J0 * 2) * 32 + lane], b01 = X[(J0 * 2 + 1) * 32 + lane];
  double b10 = 0.0, b11 = 0.0;
  if (TWO) {
    b10 = X[(J1 * 2) * 32 + lane];
    b11 = X[(J1 * 2 + 1) * 32 + lane];
  }
#pragma unroll
  for (int I = 0; I < NT; ++I) {
    const double a0 = Pf[(I * 2) * 32 + lane], a1 = Pf[(I * 2 + 1) * 32 + lane];
    dmma_ns(acc0[I][0], acc0[I][1], a0, b00);
    dmma_ns(acc0[I][0], acc0[I][1], a1, b01);
    if (TWO) {
      dmma_ns(acc1[I][0], acc1[I][1], a0, b10);
      dmma_ns(acc1[I][0], acc1[I][1], a1, b11);
    }
  }
}

template <int NT>
__host__ __device__ constexpr size_t ns_factor_rt_buf_doubles(int m) {
  // max(assembly / output matrix m x m, panel hand-over M x RT_PS + two Pf (8 M each) + X (8 M)
  // + 16 doubles of pivot-row broadcast scratch)
  return (size_t)m * m > (size_t)(RT_PS + 24) * 8 * NT + 16 ? (size_t)m * m : (size_t)(RT_PS + 24) * 8 * NT + 16;
}
template <int NT>
__host__ __device__ constexpr size_t ns_factor_rt_smem(int m, int mp) {
  return ns_factor_rt_buf_doubles<NT>(m) * sizeof(double) + (size_t)(2 * 8 * NT + mp) * sizeof(int) + 2 * 8 * NT + 16;
}

// phase timers of k_ns_factor_rt<..., PROF = true> (clock64 sums over all blocks; tools only)
__device__ unsigned long long g_rtprof[16];
#define RT_T0(v) \
  long long v = 0;   \
  if constexpr (PROF) v = clock64();
#define RT_ACC(slot, v) \
  if constexpr (PROF) \
    if (lane == 0) atomicAdd(&g_rtprof[slot], (unsigned long long)(clock64() - v));

template <int NQ, int NT, int MINB, bool PROF = false>
__global__ void __launch_bounds__(32 * ((NT + 1) / 2 + 1), MINB)
    k_ns_factor_rt(int mp, int N, int64_t mstride, const int32_t *__restrict__ pnodes, const double *__restrict__ Mv,
                   const double *__restrict__ KGv, const double *__restrict__ conv, NSTime tm,
                   double *__restrict__ out, int32_t *__restrict__ info, const int32_t *__restrict__ ppos,
                   const int32_t *__restrict__ pvv, int n0, int nwin) {
  constexpr int W = (NT + 1) / 2, M = 8 * NT;  // W accumulator warps + the panel warp (warp W)
  extern __shared__ __align__(16) double smem[];
  const int m = NQ * mp;
  double *A = smem;
  int *prow = (int *)(smem + ns_factor_rt_buf_doubles<NT>(m));
  int *qinv = prow + M;
  int *nodes = qinv + M;
  int8_t *used = (int8_t *)(nodes + mp);
  int8_t *tpos = used + M;
  __shared__ double s_red[W + 1];
  __shared__ int s_info;
  __shared__ unsigned s_pmask[16];
  const int64_t p = blockIdx.x;
  const int n = n0 + blockIdx.y;  // slab window [n0, n0 + nwin)
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5, lr = lane >> 2, lc = lane & 3;
  RT_T0(t_start)
  ns_assemble_block<NQ>(A, nodes, mp, p, n, N, pnodes, Mv, KGv, conv, tm, ppos, pvv);
  for (int r = tid; r < M; r += blockDim.x) used[r] = -1;
  if (tid == 0) s_info = 0;
  __syncthreads();
  double rn = 0.0;  // max row norm (R10 tolerance); rotated columns (no bank conflicts), 4 sums in flight
  for (int r = tid; r < m; r += blockDim.x) {
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
    const double *row = A + r * m;
    int c = r, j = 0;
    auto nx = [&](int x) { return x + 1 == m ? 0 : x + 1; };
    for (; j + 4 <= m; j += 4) {
      const int c1 = nx(c), c2 = nx(c1), c3 = nx(c2);
      s0 += fabs(row[c]);
      s1 += fabs(row[c1]);
      s2 += fabs(row[c2]);
      s3 += fabs(row[c3]);
      c = nx(c3);
    }
    for (; j < m; ++j, c = nx(c)) s0 += fabs(row[c]);
    rn = fmax(rn, (s0 + s1) + (s2 + s3));
  }
  for (int o = 16; o; o >>= 1) rn = fmax(rn, __shfl_xor_sync(0xffffffffu, rn, o));
  if (lane == 0) s_red[w] = rn;
  double *Pin = A, *Pfb = A + RT_PS * M, *X = Pfb + 16 * M;
  const int npan = (m + 7) / 8;
  // Two role loops with the same CTA barriers: the accumulators are live only in the
  // accumulator warps' loop (one shared loop would keep them live in the panel warp too).
  if (w < W) {
    double acc[2][NT][2];
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      const int J = w + W * c;
#pragma unroll
      for (int I = 0; I < NT; ++I)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int R = I * 8 + lr, C = J * 8 + 2 * lc + e;
          acc[c][I][e] = (J < NT) ? ((R < m && C < m) ? A[R * m + C] : (R == C ? 1.0 : 0.0)) : 0.0;
        }
    }
    __syncthreads();  // (1) A is free: the hand-over buffers alias it
    RT_ACC(0, t_start)
    RT_T0(t_elim)
    if (w == 0) {     // panel 0: tile column 0 handed over
#pragma unroll
      for (int I = 0; I < NT; ++I)
#pragma unroll
        for (int e = 0; e < 2; ++e) Pin[(I * 8 + lr) * RT_PS + 2 * lc + e] = acc[0][I][e];
      __syncwarp();
      asm volatile("bar.arrive 1, %0;" ::"r"(64) : "memory");
    }
    __syncthreads();  // (2) panel 0 factored
    for (int K = 0; K < npan; ++K) {
      RT_T0(t_a)
      const double *Pf = Pfb + (K & 1) * 8 * M;
      const bool next = K + 1 < npan;
      const unsigned pm = s_pmask[(K & 1) * 8 + lr];
      const int J0 = w, J1 = w + W;
      const bool v1 = J1 < NT;
      // X: the pivot rows' current values in tile column J (B-fragment order [J][h][lane]);
      // the pivot rows restart from zero (GJ: row = Pf X)
      auto xw = [&](double(&ac)[NT][2], int J) {
#pragma unroll
        for (int I = 0; I < NT; ++I)
          if ((pm >> I) & 1u) {
            const int t = tpos[I * 8 + lr];
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              X[(J * 2 + (t >> 2)) * 32 + (((2 * lc + e) << 2) | (t & 3))] = ac[I][e];
              ac[I][e] = 0.0;
            }
          }
        __syncwarp();
      };
      RT_ACC(1, t_a)
      RT_T0(t_b)
      auto take_panel = [&](double(&ac)[NT][2]) {  // the factored panel itself
#pragma unroll
        for (int I = 0; I < NT; ++I)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int t = 2 * lc + e;
            ac[I][e] = Pf[(I * 2 + (t >> 2)) * 32 + ((lr << 2) | (t & 3))];
          }
      };
      auto hand_over = [&](double(&ac)[NT][2]) {  // look-ahead column to the panel warp
#pragma unroll
        for (int I = 0; I < NT; ++I)
#pragma unroll
          for (int e = 0; e < 2; ++e) Pin[(I * 8 + lr) * RT_PS + 2 * lc + e] = ac[I][e];
        __syncwarp();
        asm volatile("bar.arrive 1, %0;" ::"r"(64) : "memory");
        RT_ACC(3, t_a)
      };
      if (J0 != K) xw(acc[0], J0);
      if (v1 && J1 != K) xw(acc[1], J1);
      if (J0 == K) {
        take_panel(acc[0]);
        if (v1) {
          rt_update<NT, false>(acc[1], acc[1], Pf, X, J1, J1, pm, lane);
          if (next && J1 == K + 1) hand_over(acc[1]);
        }
      } else if (v1 && J1 == K) {
        take_panel(acc[1]);
        rt_update<NT, false>(acc[0], acc[0], Pf, X, J0, J0, pm, lane);
        if (next && J0 == K + 1) hand_over(acc[0]);
      } else if (next && J0 == K + 1) {
        rt_update<NT, false>(acc[0], acc[0], Pf, X, J0, J0, pm, lane);
        hand_over(acc[0]);
        if (v1) rt_update<NT, false>(acc[1], acc[1], Pf, X, J1, J1, pm, lane);
      } else if (next && v1 && J1 == K + 1) {
        rt_update<NT, false>(acc[1], acc[1], Pf, X, J1, J1, pm, lane);
        hand_over(acc[1]);
        rt_update<NT, false>(acc[0], acc[0], Pf, X, J0, J0, pm, lane);
      } else if (v1) {
        rt_update<NT, true>(acc[0], acc[1], Pf, X, J0, J1, pm, lane);
      } else {
        rt_update<NT, false>(acc[0], acc[0], Pf, X, J0, J0, pm, lane);
      }
      RT_ACC(2, t_b)
      RT_T0(t_c)
      __syncthreads();
      RT_ACC(4, t_c)
    }
    RT_ACC(5, t_elim)
    // result rows to shared memory (the hand-over buffers are dead after the last barrier)
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      const int J = w + W * c;
#pragma unroll
      for (int I = 0; I < NT; ++I)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int R = I * 8 + lr, C = J * 8 + 2 * lc + e;
          if (J < NT && R < m && C < m) A[R * m + C] = acc[c][I][e];
        }
    }
  } else {
    __syncthreads();  // (1)
    double tol = 0.0;
#pragma unroll
    for (int i = 0; i <= W; ++i) tol = fmax(tol, s_red[i]);
    tol *= 1e-14;
    asm volatile("bar.sync 1, %0;" ::"r"(64) : "memory");
    rt_panel<M>(Pin, Pfb, m, 0, min(8, m), tol, prow, used, tpos, &s_info, s_pmask, X + 8 * M, lane);
    __syncthreads();  // (2)
    for (int K = 0; K < npan; ++K) {
      if (K + 1 < npan) {
        RT_T0(t_w)
        asm volatile("bar.sync 1, %0;" ::"r"(64) : "memory");
        RT_ACC(8, t_w)
        RT_T0(t_f)
        rt_panel<M>(Pin, Pfb + ((K + 1) & 1) * 8 * M, m, K + 1, min(8, m - 8 * (K + 1)), tol, prow, used, tpos,
                    &s_info, s_pmask, X + 8 * M, lane);
        RT_ACC(9, t_f)
      }
      RT_T0(t_g)
      __syncthreads();
      RT_ACC(10, t_g)
    }
  }
  RT_T0(t_o)
  __syncthreads();
  for (int c = tid; c < m; c += blockDim.x) qinv[prow[c]] = c;
  __syncthreads();
  double *o = out + (p * nwin + blockIdx.y) * mstride;  // column-major: o[sig m + rho] = D^{-1}[rho][sig]
  for (int sig = w; sig < m; sig += W + 1) {
    const int qs = qinv[sig];
    for (int rho = lane; rho < m; rho += 32) o[(int64_t)sig * m + rho] = A[prow[rho] * m + qs];
  }
  if (tid == 0) info[p * N + n] = s_info;
  RT_ACC(12, t_o)
  if constexpr (PROF)
    if (tid == 0) atomicAdd(&g_rtprof[15], 1ull);
}

// Register-tiled variant (m <= 80): thread t owns the TR x TC tile (t / NTC, t % NTC)
// of D_{p,n} in registers for the whole Gauss-Jordan; per column: (A) column c
// published, (B) pivot chosen by warp 0 (first maximum |a| among rows >= c, the
// dgetrf choice, R10), (C) the scaled pivot row and the displaced row c published;
// the update applies the interchange implicitly.  The column interchanges that
// undo the row pivoting become a permutation of the output columns; the inverse
// is written column-major for the sweep.
template <int NQ, int TR, int TC, int NTR, int NTC>
__global__ void __launch_bounds__(256) k_ns_factor_reg(int mp, int N, int64_t mstride,
                                                       const int32_t *__restrict__ pnodes,
                                                       const double *__restrict__ Mv, const double *__restrict__ KGv,
                                                       const double *__restrict__ conv, NSTime tm,
                                                       double *__restrict__ out, int32_t *__restrict__ info,
                                                       const int32_t *__restrict__ ppos,
                                                       const int32_t *__restrict__ pvv) {
  constexpr int MRP = TR * NTR, MCP = TC * NTC;
  __shared__ double colv[MRP], prow[MCP], rowc[MCP];
  __shared__ int nodes[MRP / NQ + 1], perm[MCP];
  __shared__ double s_red[8];
  __shared__ double s_pv, s_tol;
  __shared__ int s_p, s_info;
  const int m = NQ * mp;
  const int64_t p = blockIdx.x;
  const int n = blockIdx.y;
  const int64_t NT = (int64_t)N * NQ;
  const int tid = threadIdx.x, lane = tid & 31;
  const bool act = tid < NTR * NTC;
  const int tr = act ? tid / NTC : 0, tc = act ? tid % NTC : 0;
  const int R0 = tr * TR, C0 = tc * TC;
  for (int i = tid; i < mp; i += blockDim.x) nodes[i] = pnodes[p * mp + i];
  if (tid == 0) s_info = 0;
  __syncthreads();
  double A[TR][TC];
#pragma unroll
  for (int a = 0; a < TR; ++a)
#pragma unroll
    for (int b = 0; b < TC; ++b) {
      const int rho = R0 + a, sig = C0 + b;
      double v = 0.0;
      if (act && rho < m && sig < m) {
        const int i = rho / NQ, aa = rho - i * NQ, j = sig / NQ, bb = sig - j * NQ;
        if (nodes[i] < 0 || nodes[j] < 0) {
          v = (rho == sig) ? 1.0 : 0.0;
        } else {
          const int64_t e = (p * mp + i) * mp + j;
          v = block_entry_tab<NQ>(__ldg(ppos + e), __ldg(pvv + e), Mv, KGv, conv, NT, n, tm, aa, bb);
        }
      }
      A[a][b] = v;
    }
  // R10 tolerance: 1e-14 x max row sum of |D|
  {
    __shared__ double rsum[MRP][NTC + 1];
    if (act)
#pragma unroll
      for (int a = 0; a < TR; ++a) {
        double t = 0.0;
#pragma unroll
        for (int b = 0; b < TC; ++b) t += fabs(A[a][b]);
        rsum[R0 + a][tc] = t;
      }
    __syncthreads();
    double mx = 0.0;
    for (int r = tid; r < m; r += blockDim.x) {
      double t = 0.0;
      for (int b = 0; b < NTC; ++b) t += rsum[r][b];
      mx = fmax(mx, t);
    }
    for (int o = 16; o; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if (lane == 0) s_red[tid >> 5] = mx;
    __syncthreads();
    if (tid == 0) {
      double v = 0.0;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) v = fmax(v, s_red[w]);
      s_tol = 1e-14 * v;
    }
  }
  if (act && C0 == 0)
#pragma unroll
    for (int a = 0; a < TR; ++a) colv[R0 + a] = A[a][0];
  __syncthreads();  // (A)
  for (int c = 0; c < m; ++c) {
    if (tid < 32) {  // (B) pivot: first maximum |a| over rows c .. m-1
      double bv = -1.0;
      int bi = m;
      for (int r = c + lane; r < m; r += 32) {
        const double v = fabs(colv[r]);
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
        s_p = bi;
        s_pv = colv[bi];
        perm[c] = bi;
        if (!(bv >= s_tol) && s_info == 0) s_info = c + 1;
      }
    }
    __syncthreads();
    const int pr = s_p;
    const double pinv = s_pv != 0.0 ? 1.0 / s_pv : 0.0;
    const double fp = colv[c];  // multiplier of the displaced row c (it lands on row p)
    double fr[TR];              // read before (C): colv is rewritten after the update
#pragma unroll
    for (int a = 0; a < TR; ++a) fr[a] = colv[R0 + a];
    // (C) new row c = old row p / pivot (column c <- 1 / pivot); old row c kept for row p
    if (act && pr >= R0 && pr < R0 + TR)
#pragma unroll
      for (int a = 0; a < TR; ++a)
        if (R0 + a == pr)
#pragma unroll
          for (int b = 0; b < TC; ++b) prow[C0 + b] = (C0 + b == c) ? pinv : A[a][b] * pinv;
    if (act && c >= R0 && c < R0 + TR)
#pragma unroll
      for (int a = 0; a < TR; ++a)
        if (R0 + a == c)
#pragma unroll
          for (int b = 0; b < TC; ++b) rowc[C0 + b] = A[a][b];
    __syncthreads();  // (C)
    if (act) {
#pragma unroll
      for (int a = 0; a < TR; ++a) {
        const int r = R0 + a;
        if (r == c) {
#pragma unroll
          for (int b = 0; b < TC; ++b) A[a][b] = prow[C0 + b];
        } else {
          const bool isp = (r == pr);
          const double f = isp ? fp : fr[a];
#pragma unroll
          for (int b = 0; b < TC; ++b) {
            const double old = isp ? rowc[C0 + b] : A[a][b];
            A[a][b] = (C0 + b == c) ? -f * pinv : fma(-f, prow[C0 + b], old);
          }
        }
      }
      if (c + 1 < m && c + 1 >= C0 && c + 1 < C0 + TC)  // publish column c + 1
#pragma unroll
        for (int b = 0; b < TC; ++b)
          if (C0 + b == c + 1)
#pragma unroll
            for (int a = 0; a < TR; ++a) colv[R0 + a] = A[a][b];
    }
    __syncthreads();  // (A)
  }
  // (P A)^{-1} = A^{-1} P^T: arr[pos] = work column at final position pos; dstc = arr^-1
  __shared__ int arr[MCP], dstc[MCP];
  if (tid == 0) {
    for (int j = 0; j < m; ++j) arr[j] = j;
    for (int c = m - 1; c >= 0; --c) {
      const int pc = perm[c];
      if (pc != c) {
        const int t = arr[c];
        arr[c] = arr[pc];
        arr[pc] = t;
      }
    }
    for (int j = 0; j < m; ++j) dstc[arr[j]] = j;
  }
  __syncthreads();
  double *o = out + (p * N + n) * mstride;  // column-major: o[sig m + rho] = D^{-1}[rho][sig]
  if (act)
#pragma unroll
    for (int b = 0; b < TC; ++b) {
      const int sig = C0 + b;
      if (sig >= m) continue;
      const int dst = dstc[sig];
#pragma unroll
      for (int a = 0; a < TR; ++a)
        if (R0 + a < m) o[(int64_t)dst * m + R0 + a] = A[a][b];
    }
  if (tid == 0) info[p * N + n] = s_info;
}

// Row-per-thread Gauss-Jordan (m <= MMAX): thread r holds row r of D_{p,n} in
// registers.  Step c: the unused row with the largest |a[c]| (first such row on
// ties: partial pivoting, R10) is scaled and broadcast through shared memory,
// every other row eliminates column c in place (implicit pivoting: no row moves).
// With p_c the pivot row of step c, the in-place result X gives
//     D^{-1}[c][p_k] = X[p_c][k],
// written column-major for the sweep.  Two barriers per step, no dynamic register
// indexing (a[c] is picked by a predicated select over the unrolled row).
template <int NQ, int MMAX, int NTH>
__global__ void __launch_bounds__(NTH) k_ns_factor_row(int mp, int N, int64_t mstride,
                                                        const int32_t *__restrict__ pnodes,
                                                        const double *__restrict__ Mv,
                                                        const double *__restrict__ KGv,
                                                        const double *__restrict__ conv, NSTime tm,
                                                        double *__restrict__ out, int32_t *__restrict__ info,
                                                        const int32_t *__restrict__ ppos,
                                                        const int32_t *__restrict__ pvv) {
  __shared__ __align__(16) double prow[MMAX];
  __shared__ int nodes[MMAX / NQ + 1], pcs[MMAX];
  __shared__ double s_wv[2 * (NTH / 32)];
  __shared__ int s_wi[2 * (NTH / 32)];
  __shared__ double s_tol, s_pv;
  __shared__ int s_info;
  const int m = NQ * mp;
  const int64_t p = blockIdx.x;
  const int n = blockIdx.y;
  const int64_t NT = (int64_t)N * NQ;
  const int r = threadIdx.x, lane = r & 31, w = r >> 5;
  constexpr int NW = NTH / 32;
  for (int i = r; i < mp; i += NTH) nodes[i] = pnodes[p * mp + i];
  if (r == 0) s_info = 0;
  __syncthreads();
  const bool live = r < m;
  double a[MMAX];
  {
    const int i = r / NQ, ar = r - (r / NQ) * NQ;
    const bool rowpad = !live || nodes[live ? i : 0] < 0;
#pragma unroll
    for (int j = 0; j < MMAX; ++j) {
      double v = 0.0;
      if (live && j < m) {
        const int jn = j / NQ, bb = j - jn * NQ;
        if (rowpad || nodes[jn] < 0) {
          v = (r == j) ? 1.0 : 0.0;
        } else {
          const int64_t e = (p * mp + i) * mp + jn;
          v = block_entry_tab<NQ>(__ldg(ppos + e), __ldg(pvv + e), Mv, KGv, conv, NT, n, tm, ar, bb);
        }
      }
      a[j] = v;
    }
  }
  {  // R10 tolerance: 1e-14 x max row sum
    double rs = 0.0;
#pragma unroll
    for (int j = 0; j < MMAX; ++j) rs += fabs(a[j]);
    for (int o = 16; o; o >>= 1) rs = fmax(rs, __shfl_xor_sync(0xffffffffu, rs, o));
    if (lane == 0) s_wv[w] = rs;
    __syncthreads();
    if (r == 0) {
      double mx = 0.0;
      for (int k = 0; k < NW; ++k) mx = fmax(mx, s_wv[k]);
      s_tol = 1e-14 * mx;
    }
    __syncthreads();
  }
  bool used = !live;
  int mystep = -1;
  // Steps in blocks of 8 columns: inside a block the column index is static, the
  // block index cb is a runtime loop (compact code).  The block's 8 columns live in
  // blk[] (extracted / written back by selects over cb); the full-row update also
  // touches the stale copy a[cb][.], which the write-back overwrites.
  constexpr int NB = MMAX / 8;
  const int nb = (m + 7) / 8;
  for (int cb = 0; cb < nb; ++cb) {
    double blk[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      double v = 0.0;
#pragma unroll
      for (int b2 = 0; b2 < NB; ++b2) v = (b2 == cb) ? a[b2 * 8 + k] : v;
      blk[k] = v;
    }
#pragma unroll 1
    for (int k = 0; k < 8; ++k) {  // runtime step loop: the body (~400 instructions) stays in the I-cache
      const int c = cb * 8 + k;
      if (c < m) {
        double ac = 0.0;
#pragma unroll
        for (int k2 = 0; k2 < 8; ++k2) ac = (k2 == k) ? blk[k2] : ac;
        double bv = used ? -1.0 : fabs(ac);
        int bi = used ? NTH : r;
        for (int o = 16; o; o >>= 1) {
          const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
          const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
          if (ov > bv || (ov == bv && oi < bi)) {
            bv = ov;
            bi = oi;
          }
        }
        // per-warp maxima; every thread combines them itself (no second barrier).
        // Double-buffered by step parity: a fast warp may publish step c+1 while a
        // slow one still reads step c.
        if (lane == 0) {
          s_wv[(c & 1) * NW + w] = bv;
          s_wi[(c & 1) * NW + w] = bi;
        }
        __syncthreads();
        double pv = s_wv[(c & 1) * NW];
        int pr = s_wi[(c & 1) * NW];
#pragma unroll
        for (int k2 = 1; k2 < NW; ++k2) {
          const double v2 = s_wv[(c & 1) * NW + k2];
          const int i2 = s_wi[(c & 1) * NW + k2];
          if (v2 > pv || (v2 == pv && i2 < pr)) {
            pv = v2;
            pr = i2;
          }
        }
        if (r == 0) {
          pcs[c] = pr;
          if (!(pv >= s_tol) && s_info == 0) s_info = c + 1;
        }
        if (r == pr) {  // publish the raw pivot row (block columns from blk) and the pivot
#pragma unroll
          for (int j = 0; j < MMAX; j += 2) *reinterpret_cast<double2 *>(prow + j) = make_double2(a[j], a[j + 1]);
#pragma unroll
          for (int k2 = 0; k2 < 8; ++k2) prow[cb * 8 + k2] = blk[k2];
          s_pv = ac;
        }
        __syncthreads();
        const double piv = s_pv, pinv = piv != 0.0 ? 1.0 / piv : 0.0;
        if (r == pr) {  // pivot row: column c <- 1, then scale (column c becomes 1 / pivot)
#pragma unroll
          for (int j = 0; j < MMAX; ++j) a[j] *= pinv;
#pragma unroll
          for (int k2 = 0; k2 < 8; ++k2) blk[k2] = (k2 == k) ? pinv : blk[k2] * pinv;
          used = true;
          mystep = c;
        } else if (live) {  // eliminate with the raw pivot row: f / pivot folded into the multiplier
          const double fs = ac * pinv;
#pragma unroll
          for (int j = 0; j < MMAX; j += 2) {
            const double2 pw = *reinterpret_cast<const double2 *>(prow + j);
            a[j] = fma(-fs, pw.x, a[j]);
            a[j + 1] = fma(-fs, pw.y, a[j + 1]);
          }
#pragma unroll
          for (int k2 = 0; k2 < 8; ++k2) blk[k2] = (k2 == k) ? -fs : fma(-fs, prow[cb * 8 + k2], blk[k2]);
        }
        // prow is rewritten only after the next step's first barrier
      }
    }
#pragma unroll
    for (int k = 0; k < 8; ++k)
#pragma unroll
      for (int b2 = 0; b2 < NB; ++b2)
        if (b2 == cb) a[b2 * 8 + k] = blk[k];
  }
  __syncthreads();
  double *o = out + (p * N + n) * mstride;  // column-major: o[sig m + rho] = D^{-1}[rho][sig]
  if (live)
#pragma unroll
    for (int k = 0; k < MMAX; ++k)
      if (k < m) o[(int64_t)pcs[k] * m + mystep] = a[k];
  if (r == 0) info[p * N + n] = s_info;
}

// ---------------------------------------------------------------- H7 + H8 sweep
__device__ __forceinline__ void mbar_init_ns(uint64_t *bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"((unsigned)__cvta_generic_to_shared(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_wait_ns(uint64_t *bar, unsigned parity) {
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
// 1D TMA bulk copy global -> shared, completion on the mbarrier (bytes % 16 == 0).
__device__ __forceinline__ void bulk_load(void *dst, const void *src, unsigned bytes, uint64_t *bar) {
  const unsigned b = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(b), "r"(bytes) : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          (unsigned)__cvta_generic_to_shared(dst)),
      "l"(src), "r"(bytes), "r"(b)
      : "memory");
}

// One CTA per patch; slabs in order.  x_n = D_{p,n}^{-1} (r_{p,n} + [a = 0] M_p x_{n-1}[q]),
// u += omega W_p x (R11).  STAGED: D^{-1} of slab n+1 is bulk-copied into the other
// half of a shared double buffer while slab n is solved.
template <int NQ, bool STAGED>
__global__ void __launch_bounds__(256) k_ns_sweep(int mp, int N, int64_t mstride, const int32_t *__restrict__ pnodes,
                                                  const double *__restrict__ wnode, const int32_t *__restrict__ rowptr,
                                                  const int32_t *__restrict__ col, const double *__restrict__ Mv,
                                                  const double *__restrict__ Dinv, const double *__restrict__ r,
                                                  double *__restrict__ u, double omega, int n0, int nwin,
                                                  double *__restrict__ xs) {
  extern __shared__ __align__(128) double smem[];
  __shared__ __align__(8) uint64_t bar[2];
  const int m = NQ * mp;
  double *buf = smem;                                   // STAGED: 2 x mstride
  double *Mp = smem + (STAGED ? 2 * mstride : 0);       // mp x mp velocity mass of the patch
  const int MR = (m + 31) & ~31, G = blockDim.x / MR;  // matvec: MR rows x G column groups
  double *g = Mp + mp * mp, *x = g + m, *xq = x + m, *wn = xq + mp, *part = wn + mp;
  int *nodes = (int *)(part + 256);
  const int64_t p = blockIdx.x;
  const int64_t NT = (int64_t)N * NQ;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, nw = blockDim.x >> 5;
  // slab window [n0, n0 + nwin): Dinv holds the window's inverses, xs (windows after the
  // first) the patch solution of slab n0 - 1 for the jump
  const double *Dp = Dinv + p * nwin * mstride;
  const unsigned bytes = (unsigned)(m * m * sizeof(double) + 15) & ~15u;
  if (STAGED && tid == 0) {
    mbar_init_ns(&bar[0], 1);
    mbar_init_ns(&bar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    bulk_load(buf, Dp, bytes, &bar[0]);
  }
  for (int i = tid; i < mp; i += blockDim.x) {
    const int s = pnodes[p * mp + i];
    nodes[i] = s;
    wn[i] = s >= 0 ? omega * wnode[s] : 0.0;
    xq[i] = 0.0;
  }
  for (int i = tid; i < m; i += blockDim.x) x[i] = (n0 > 0 && xs) ? xs[p * m + i] : 0.0;
  __syncthreads();
  for (int e = tid; e < mp * mp; e += blockDim.x) {
    const int i = e / mp, j = e - i * mp;
    double v = 0.0;
    if (nodes[i] >= 0 && nodes[j] >= 0) {
      const int pos = csr_find_ns(rowptr, col, nodes[i], nodes[j]);
      if (pos >= 0) v = Mv[pos];
    }
    Mp[e] = v;
  }
  __syncthreads();
  // thread rho < m owns row rho of the patch system (m <= blockDim, checked by the launcher);
  // the r gather of slab n+1 is issued while slab n is solved
  const int i_me = tid / NQ, a_me = tid - (tid / NQ) * NQ;
  const bool own = tid < m && nodes[i_me < mp ? i_me : 0] >= 0 && i_me < mp;
  const int64_t rbase = own ? (int64_t)nodes[i_me] * NT + a_me : 0;
  const int n1 = n0 + nwin;
  double rcur = own ? __ldg(r + rbase + (int64_t)n0 * NQ) : 0.0;
  for (int n = n0; n < n1; ++n) {
    const int ln = n - n0;  // slab within the window
    if (STAGED && tid == 0 && n + 1 < n1) {
      asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
      bulk_load(buf + ((ln + 1) & 1) * mstride, Dp + (int64_t)(ln + 1) * mstride, bytes, &bar[(ln + 1) & 1]);
    }
    const double rnext = (own && n + 1 < n1) ? __ldg(r + rbase + (int64_t)(n + 1) * NQ) : 0.0;
    if (tid < m) {
      double v = rcur;
      if (own && a_me == 0 && n > 0)  // jump: M_p x_{n-1}[q] (x still holds slab n-1)
        for (int j = 0; j < mp; ++j) v = fma(Mp[i_me * mp + j], x[j * NQ + NQ - 1], v);
      g[tid] = v;
    }
    rcur = rnext;
    __syncthreads();
    const double *D;
    if (STAGED) {
      mbar_wait_ns(&bar[ln & 1], (ln >> 1) & 1);
      D = buf + (ln & 1) * mstride;
    } else {
      D = Dp + (int64_t)ln * mstride;
    }
    // x = D^{-1} g with D^{-1} column-major: thread (rho, grp) sums columns
    // sig = grp, grp + G, ... (consecutive rho -> consecutive banks), partials in smem
    {
      const int rho = tid % MR, grp = tid / MR;
      double acc = 0.0;
      if (rho < m && grp < G)
        for (int s2 = grp; s2 < m; s2 += G)
          acc = fma(STAGED ? D[s2 * m + rho] : __ldg(D + (int64_t)s2 * m + rho), g[s2], acc);
      if (grp < G) part[grp * MR + rho] = acc;
    }
    __syncthreads();
    if (tid < m) {
      double xv = 0.0;
      for (int g2 = 0; g2 < G; ++g2) xv += part[g2 * MR + tid];
      x[tid] = xv;
      if (own) atomicAdd(u + rbase + (int64_t)n * NQ, wn[i_me] * xv);
    }
    __syncthreads();
  }
  if (xs && n1 < N)
    for (int i = tid; i < m; i += blockDim.x) xs[p * m + i] = x[i];
}

// Large blocks (m x m too big for a shared double buffer, e.g. P3-P2 x DG1,
// m = 162): D^{-1} of each slab streamed in chunks of CW columns (contiguous in
// the column-major layout) through a ring of R shared slots by 1-D TMA bulk
// copies; the ring runs ahead across slab boundaries (D_{p,n+1} does not depend
// on x_n), so the stream never drains inside a patch.  Thread rho < m owns row rho.
template <int NQ>
__global__ void __launch_bounds__(256) k_ns_sweep_chunked(int mp, int N, int64_t mstride, int CW, int R,
                                                          const int32_t *__restrict__ pnodes,
                                                          const double *__restrict__ wnode,
                                                          const int32_t *__restrict__ rowptr,
                                                          const int32_t *__restrict__ col,
                                                          const double *__restrict__ Mv,
                                                          const double *__restrict__ Dinv, const double *__restrict__ r,
                                                          double *__restrict__ u, double omega, int n0, int nwin,
                                                          double *__restrict__ xs) {
  extern __shared__ __align__(128) double smem[];
  __shared__ __align__(8) uint64_t bar[8];
  const int m = NQ * mp;
  const int64_t slot = (int64_t)CW * m;                 // doubles per ring slot
  double *ring = smem;                                  // R x slot
  double *Mp = smem + R * slot;                         // mp x mp velocity mass of the patch
  double *g = Mp + mp * mp, *x = g + m, *wn = x + m;
  int *nodes = (int *)(wn + mp);
  const int64_t p = blockIdx.x;
  const int64_t NT = (int64_t)N * NQ;
  const int tid = threadIdx.x;
  const double *Dp = Dinv + p * nwin * mstride;  // the window [n0, n0 + nwin) (k_ns_sweep)
  const int nch = (m + CW - 1) / CW;
  const int64_t total = (int64_t)nwin * nch;
  auto issue = [&](int64_t t) {  // chunk t = (slab n, chunk c) into slot t % R
    const int64_t n = t / nch;
    const int c = (int)(t - n * nch);
    const int cols = min(CW, m - c * CW);
    const unsigned bytes = (unsigned)((int64_t)cols * m * sizeof(double) + 15) & ~15u;
    bulk_load(ring + (t % R) * slot, Dp + n * mstride + (int64_t)c * CW * m, bytes, &bar[t % R]);
  };
  if (tid == 0) {
    for (int k = 0; k < R; ++k) mbar_init_ns(&bar[k], 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    for (int64_t t = 0; t < R && t < total; ++t) issue(t);
  }
  for (int i = tid; i < mp; i += blockDim.x) {
    const int sn = pnodes[p * mp + i];
    nodes[i] = sn;
    wn[i] = sn >= 0 ? omega * wnode[sn] : 0.0;
  }
  __syncthreads();
  for (int e = tid; e < mp * mp; e += blockDim.x) {
    const int i = e / mp, j = e - i * mp;
    double v = 0.0;
    if (nodes[i] >= 0 && nodes[j] >= 0) {
      const int pos = csr_find_ns(rowptr, col, nodes[i], nodes[j]);
      if (pos >= 0) v = Mv[pos];
    }
    Mp[e] = v;
  }
  for (int i = tid; i < m; i += blockDim.x) x[i] = (n0 > 0 && xs) ? xs[p * m + i] : 0.0;
  __syncthreads();
  const int i_me = tid / NQ, a_me = tid - (tid / NQ) * NQ;
  const bool own = tid < m && i_me < mp && nodes[i_me] >= 0;
  const int64_t rbase = own ? (int64_t)nodes[i_me] * NT + a_me : 0;
  const int n1 = n0 + nwin;
  double rcur = own ? __ldg(r + rbase + (int64_t)n0 * NQ) : 0.0;
  for (int n = n0; n < n1; ++n) {
    const double rnext = (own && n + 1 < n1) ? __ldg(r + rbase + (int64_t)(n + 1) * NQ) : 0.0;
    if (tid < m) {
      double v = rcur;
      if (own && a_me == 0 && n > 0)  // jump: M_p x_{n-1}[q]
        for (int j = 0; j < mp; ++j) v = fma(Mp[i_me * mp + j], x[j * NQ + NQ - 1], v);
      g[tid] = v;
    }
    rcur = rnext;
    __syncthreads();
    double acc = 0.0;
    for (int c = 0; c < nch; ++c) {
      const int64_t t = (int64_t)(n - n0) * nch + c;
      mbar_wait_ns(&bar[t % R], (unsigned)((t / R) & 1));
      const double *D = ring + (t % R) * slot;
      const int cols = min(CW, m - c * CW);
      if (tid < m) {
        const double *gc = g + c * CW;
        for (int j = 0; j < cols; ++j) acc = fma(D[j * m + tid], gc[j], acc);
      }
      __syncthreads();  // slot consumed by every thread
      if (tid == 0 && t + R < total) {
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        issue(t + R);
      }
    }
    if (tid < m) {
      x[tid] = acc;
      if (own) atomicAdd(u + rbase + (int64_t)n * NQ, wn[i_me] * acc);
    }
    __syncthreads();
  }
  if (xs && n1 < N)
    for (int i = tid; i < m; i += blockDim.x) xs[p * m + i] = x[i];
}

// --------------------------------------------------------------- H15 projection
// partial[b][t] = sum of rows [b*rpb, (b+1)*rpb) of the Lp x NT pressure block.
__global__ void k_colsum(const double *__restrict__ P, int64_t nrow, int64_t NT, int64_t rpb,
                         double *__restrict__ partial) {
  const int64_t r0 = blockIdx.x * rpb, r1 = min(nrow, r0 + rpb);
  for (int64_t t = threadIdx.x; t < NT; t += blockDim.x) {
    double s = 0.0;
    for (int64_t rr = r0; rr < r1; ++rr) s += P[rr * NT + t];
    partial[blockIdx.x * NT + t] = s;
  }
}
__global__ void k_colmean(const double *__restrict__ partial, int nb, int64_t NT, int64_t nrow, double *__restrict__ mean) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < NT; t += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int b = 0; b < nb; ++b) s += partial[(int64_t)b * NT + t];
    mean[t] = s / (double)nrow;
  }
}
__global__ void k_colsub(double *__restrict__ P, int64_t nrow, int64_t NT, const double *__restrict__ mean) {
  const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (idx >= nrow * NT) return;
  P[idx] -= mean[idx % NT];
}

// ------------------------------------------------------------------ H11 coarse
// Column-major block of slab n over the free coarse sids; the rows of the pinned
// pressure DoF (first pressure node, every temporal node) are identity rows (R19).
template <int NQ>
__global__ void k_ns_coarse_blocks(int mc, int N, int pin, const int32_t *__restrict__ cnodes,
                                   const int32_t *__restrict__ rowptr, const int32_t *__restrict__ col,
                                   const double *__restrict__ Mv, const double *__restrict__ KGv, int64_t nvrow,
                                   const int32_t *__restrict__ vvptr, const double *__restrict__ conv, NSTime tm,
                                   double *__restrict__ D) {
  const int n = blockIdx.y;
  const int64_t m = (int64_t)NQ * mc, NT = (int64_t)N * NQ;
  double *Dn = D + (int64_t)n * m * m;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m * m; e += (int64_t)gridDim.x * blockDim.x) {
    const int sig = (int)(e / m), rho = (int)(e - (int64_t)sig * m);
    const int i = rho / NQ, a = rho - i * NQ, j = sig / NQ, bb = sig - j * NQ;
    double v;
    if (i == pin)
      v = (rho == sig) ? 1.0 : 0.0;
    else
      v = block_entry<NQ>(rowptr, col, Mv, KGv, nvrow, vvptr, conv, NT, n, tm, cnodes[i], cnodes[j], a, bb);
    Dn[e] = v;
  }
}

// Block forward substitution over slabs (one CTA): g = r_n + [a=0] M x_{n-1}[q]
// (pinned rows 0), x_n = D_n^{-1} g; z receives x on free sids (z pre-zeroed).
template <int NQ>
__global__ void __launch_bounds__(1024) k_ns_coarse_solve(int mc, int N, int pin, const int32_t *__restrict__ cnodes,
                                                          const int32_t *__restrict__ rowptr,
                                                          const int32_t *__restrict__ col,
                                                          const double *__restrict__ Mv,
                                                          const double *__restrict__ DinvT, const double *__restrict__ r,
                                                          double *__restrict__ z, double *__restrict__ xq) {
  extern __shared__ double sm[];
  const int m = NQ * mc;
  double *g = sm;
  const int64_t NT = (int64_t)N * NQ;
  const int tid = threadIdx.x;
  for (int n = 0; n < N; ++n) {
    for (int rho = tid; rho < m; rho += blockDim.x) {
      const int i = rho / NQ, a = rho - i * NQ;
      const int s = cnodes[i];
      double v = 0.0;
      if (i != pin) {
        v = r[(int64_t)s * NT + (int64_t)n * NQ + a];
        if (a == 0 && n > 0)
          for (int e = rowptr[s]; e < rowptr[s + 1]; ++e) v = fma(Mv[e], xq[col[e]], v);
      }
      g[rho] = v;
    }
    __syncthreads();
    const double *Di = DinvT + (int64_t)n * m * m;
    double xv[2] = {0.0, 0.0};
    for (int k2 = 0; k2 < 2; ++k2) {
      const int rho = tid + k2 * blockDim.x;
      if (rho >= m) break;
      double acc = 0.0;
      for (int s2 = 0; s2 < m; ++s2) acc = fma(Di[(int64_t)s2 * m + rho], g[s2], acc);
      xv[k2] = acc;
    }
    __syncthreads();  // every thread has read xq of slab n-1 (through g)
    for (int k2 = 0; k2 < 2; ++k2) {
      const int rho = tid + k2 * blockDim.x;
      if (rho >= m) break;
      const int i = rho / NQ, a = rho - i * NQ;
      const int s = cnodes[i];
      z[(int64_t)s * NT + (int64_t)n * NQ + a] = xv[k2];
      if (a == NQ - 1) xq[s] = xv[k2];
    }
    __syncthreads();
  }
}

// ---- Parallel-in-time coarse march.  With E the jump (rows (i, a=0) of free sid i:
// E[(i,0), j] = M[s_i, s_j], pinned row 0) and y_n = x_n[a = q] (per free sid):
//   x_n = D_n^{-1} r_n + H_n y_{n-1},  H_n = D_n^{-1} E,   y_n = x_n[q] = z_n[q] + G_n y_{n-1}
// (G_n = the a = q rows of H_n).  H_n and G_n are formed once per linearisation;
// a solve is then two slab-parallel GEMV passes around an mp-sized recurrence.
// H[(n mp + j) m + rho] = sum_{e in row(s_j)} M_e D_n^{-1}[rho][(idx(col_e), 0)]  (M symmetric)
template <int NQ>
__global__ void k_ns_coarse_H(int mc, int N, int pin, const int32_t *__restrict__ cnodes,
                              const int32_t *__restrict__ sid2c, const int32_t *__restrict__ rowptr,
                              const int32_t *__restrict__ col, const double *__restrict__ Mv,
                              const double *__restrict__ DinvT, double *__restrict__ H, double *__restrict__ G) {
  const int m = NQ * mc;
  const int rho = blockIdx.x * blockDim.x + threadIdx.x, j = blockIdx.y, n = blockIdx.z;
  if (rho >= m) return;
  const double *Di = DinvT + (int64_t)n * m * m;
  const int sj = cnodes[j];
  double acc = 0.0;
  for (int e = rowptr[sj]; e < rowptr[sj + 1]; ++e) {
    const int i = sid2c[col[e]];
    if (i >= 0 && i != pin) acc = fma(Mv[e], Di[(int64_t)(i * NQ) * m + rho], acc);
  }
  H[((int64_t)n * mc + j) * m + rho] = acc;
  if (rho % NQ == NQ - 1) G[((int64_t)n * mc + j) * mc + rho / NQ] = acc;
}

// z_n = D_n^{-1} r_n (pinned row of r taken as 0): CTA = (slab, 32 rows), warp w
// sums columns w, w + 8, ...; out[n m + rho].  With H (K3) the CTA adds H_n y_{n-1}
// and scatters x_n to the sid layout.
template <int NQ, bool FINAL>
__global__ void __launch_bounds__(256) k_ns_coarse_pass(int mc, int N, int pin, const int32_t *__restrict__ cnodes,
                                                        const double *__restrict__ DinvT,
                                                        const double *__restrict__ r, double *__restrict__ Z,
                                                        const double *__restrict__ H, const double *__restrict__ Y,
                                                        double *__restrict__ z) {
  extern __shared__ double gsh[];  // m (pass 1) or mc (pass 2)
  __shared__ double part[8][33];
  const int m = NQ * mc, n = blockIdx.x, rb = blockIdx.y * 32;
  const int tid = threadIdx.x, rl = tid & 31, w = tid >> 5;
  const int64_t NT = (int64_t)N * NQ;
  double acc = 0.0;
  const int rho = rb + rl;
  if (!FINAL) {
    for (int s2 = tid; s2 < m; s2 += blockDim.x) {
      const int i = s2 / NQ, a = s2 - i * NQ;
      gsh[s2] = (i != pin) ? __ldg(r + (int64_t)cnodes[i] * NT + (int64_t)n * NQ + a) : 0.0;
    }
    __syncthreads();
    if (rho < m) {
      const double *Di = DinvT + (int64_t)n * m * m;
      for (int s2 = w; s2 < m; s2 += 8) acc = fma(__ldg(Di + (int64_t)s2 * m + rho), gsh[s2], acc);
    }
  } else {
    if (n > 0) {
      for (int j = tid; j < mc; j += blockDim.x) gsh[j] = Y[(int64_t)(n - 1) * mc + j];
      __syncthreads();
      if (rho < m) {
        const double *Hn = H + (int64_t)n * mc * m;
        for (int j = w; j < mc; j += 8) acc = fma(__ldg(Hn + (int64_t)j * m + rho), gsh[j], acc);
      }
    }
  }
  part[w][rl] = acc;
  __syncthreads();
  if (w == 0 && rho < m) {
    double t = 0.0;
#pragma unroll
    for (int k = 0; k < 8; ++k) t += part[k][rl];
    if (!FINAL) {
      Z[(int64_t)n * m + rho] = t;
    } else {
      const int i = rho / NQ, a = rho - i * NQ;
      z[(int64_t)cnodes[i] * NT + (int64_t)n * NQ + a] = Z[(int64_t)n * m + rho] + t;
    }
  }
}

// y_n = z_n[q] + G_n y_{n-1} (y_{-1} = 0), one CTA of 1024 threads: thread (row
// jj = t % R + R k, column group t / R of CG, R = 1024 / CG); y double-buffered by
// slab parity, two barriers per slab; Y[n mp + jj].  Shared memory (2 + CG) mc
// doubles: CG = 8, or 2 for the largest coarse levels (mc > 2560).
template <int NQ, int CG>
__global__ void __launch_bounds__(1024) k_ns_coarse_yrec(int mc, int N, const double *__restrict__ Z,
                                                         const double *__restrict__ G, double *__restrict__ Y) {
  extern __shared__ double sh[];  // y (2 mc) + partials (CG mc)
  constexpr int R = 1024 / CG;
  double *yb = sh, *pp = sh + 2 * mc;
  const int m = NQ * mc, tid = threadIdx.x, rr = tid % R, cg = tid / R;
  for (int j = tid; j < 2 * mc; j += blockDim.x) yb[j] = 0.0;
  __syncthreads();
  for (int n = 0; n < N; ++n) {
    const double *Gn = G + (int64_t)n * mc * mc;
    const double *yp = yb + ((n + 1) & 1) * mc;
    double *yn = yb + (n & 1) * mc;
    for (int jj = rr; jj < mc; jj += R) {
      double a0 = 0.0, a1 = 0.0;
      if (n > 0) {
        int j = cg;
        for (; j + CG < mc; j += 2 * CG) {
          a0 = fma(__ldg(Gn + (int64_t)j * mc + jj), yp[j], a0);
          a1 = fma(__ldg(Gn + (int64_t)(j + CG) * mc + jj), yp[j + CG], a1);
        }
        if (j < mc) a0 = fma(__ldg(Gn + (int64_t)j * mc + jj), yp[j], a0);
      }
      pp[cg * mc + jj] = a0 + a1;
    }
    __syncthreads();
    for (int jj = tid; jj < mc; jj += blockDim.x) {
      double v = Z[(int64_t)n * m + jj * NQ + NQ - 1];
#pragma unroll
      for (int k = 0; k < CG; ++k) v += pp[k * mc + jj];
      yn[jj] = v;
      Y[(int64_t)n * mc + jj] = v;
    }
    __syncthreads();
  }
}

// Cluster variant: CS CTAs share the slab loop; CTA c owns rows [c RB, (c+1) RB)
// of every D_n^{-1} (RB = ceil(m / CS)), every CTA forms the full g (the jump needs
// the whole end trace, kept per sid in each CTA's shared memory and broadcast
// through distributed shared memory), one cluster barrier per slab.
template <int NQ, int CS>
__global__ void __cluster_dims__(CS, 1, 1) __launch_bounds__(256)
    k_ns_coarse_cluster(int mc, int N, int pin, int64_t ns, const int32_t *__restrict__ cnodes,
                        const int32_t *__restrict__ rowptr, const int32_t *__restrict__ col,
                        const double *__restrict__ Mv, const double *__restrict__ DinvT,
                        const double *__restrict__ r, double *__restrict__ z, int nnzj) {
  namespace cg = cooperative_groups;
  cg::cluster_group cluster = cg::this_cluster();
  extern __shared__ double sm[];
  const int m = NQ * mc;
  // xq: end trace per sid, double-buffered by slab parity (a CTA may publish slab n
  // while another still reads slab n-1 for its g); 0 on constrained sids.
  // The mass rows of the jump are staged once in shared memory (jp / jc / jv).
  double *g = sm, *xqb = sm + m, *jv = xqb + 2 * ns;
  int *jc = reinterpret_cast<int *>(jv + nnzj), *jp = jc + nnzj;
  __shared__ double part[8][33];
  const int64_t NT = (int64_t)N * NQ;
  const int tid = threadIdx.x, rl = tid & 31, grp = tid >> 5;
  const int rank = (int)cluster.block_rank();
  const int RB = (m + CS - 1) / CS, r0 = rank * RB, r1 = min(m, r0 + RB);
  for (int64_t s = tid; s < 2 * ns; s += blockDim.x) xqb[s] = 0.0;
  if (tid == 0) {
    int acc = 0;
    for (int i = 0; i < mc; ++i) {
      jp[i] = acc;
      acc += rowptr[cnodes[i] + 1] - rowptr[cnodes[i]];
    }
    jp[mc] = acc;
  }
  __syncthreads();
  for (int i = grp; i < mc; i += blockDim.x >> 5) {
    const int s = cnodes[i], e0 = rowptr[s], ne = rowptr[s + 1] - e0;
    for (int e = rl; e < ne; e += 32) {
      jc[jp[i] + e] = col[e0 + e];
      jv[jp[i] + e] = Mv[e0 + e];
    }
  }
  // r of slab 0 (thread rho < m; m <= 2 * blockDim checked by the launcher)
  double rn[2] = {0.0, 0.0};
  for (int k2 = 0; k2 < 2; ++k2) {
    const int rho = tid + k2 * blockDim.x;
    if (rho < m) {
      const int i = rho / NQ, a = rho - i * NQ;
      if (i != pin) rn[k2] = __ldg(r + (int64_t)cnodes[i] * NT + a);
    }
  }
  cluster.sync();
  for (int n = 0; n < N; ++n) {
    const double *xq = xqb + ((n + 1) & 1) * ns;  // slab n-1
    double *xo = xqb + (n & 1) * ns;              // slab n
    for (int k2 = 0; k2 < 2; ++k2) {
      const int rho = tid + k2 * blockDim.x;
      if (rho >= m) break;
      const int i = rho / NQ, a = rho - i * NQ;
      double v = rn[k2];
      if (i != pin) {
        if (n + 1 < N) rn[k2] = __ldg(r + (int64_t)cnodes[i] * NT + (int64_t)(n + 1) * NQ + a);  // next slab
        if (a == 0 && n > 0)
          for (int e = jp[i]; e < jp[i + 1]; ++e) v = fma(jv[e], xq[jc[e]], v);
      }
      g[rho] = v;
    }
    __syncthreads();
    const double *Di = DinvT + (int64_t)n * m * m;
    for (int rb = r0; rb < r1; rb += 32) {
      const int rho = rb + rl;
      double acc = 0.0;
      if (rho < r1) {
        // 8 independent loads in flight per thread (the slab loop is latency-bound)
        double a8[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        int s2 = grp;
        for (; s2 + 56 < m; s2 += 64) {
          double v[8];
#pragma unroll
          for (int u2 = 0; u2 < 8; ++u2) v[u2] = __ldg(Di + (int64_t)(s2 + 8 * u2) * m + rho);
#pragma unroll
          for (int u2 = 0; u2 < 8; ++u2) a8[u2] = fma(v[u2], g[s2 + 8 * u2], a8[u2]);
        }
        for (; s2 < m; s2 += 8) a8[0] = fma(__ldg(Di + (int64_t)s2 * m + rho), g[s2], a8[0]);
#pragma unroll
        for (int u2 = 0; u2 < 8; ++u2) acc += a8[u2];
      }
      part[grp][rl] = acc;
      __syncthreads();
      if (grp == 0 && rho < r1) {
        double x = 0.0;
#pragma unroll
        for (int k2 = 0; k2 < 8; ++k2) x += part[k2][rl];
        const int i = rho / NQ, a = rho - i * NQ;
        const int s = cnodes[i];
        z[(int64_t)s * NT + (int64_t)n * NQ + a] = x;
        if (a == NQ - 1)
          for (int c = 0; c < CS; ++c) *cluster.map_shared_rank(xo + s, c) = x;
      }
      __syncthreads();
    }
    cluster.sync();
  }
}

// dst = src on free sids; g[s] (or 0) on constrained sids (R5, R6).
// dst = boundary value on constrained sids (gst: per space-time DoF, else g: per
// sid, else 0), src (or 0) on free sids
__global__ void k_ns_mask(int64_t ns, int64_t NT, const uint8_t *__restrict__ con, const double *__restrict__ g,
                          const double *__restrict__ gst, const double *__restrict__ src, double *__restrict__ dst) {
  const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (idx >= ns * NT) return;
  const int64_t s = idx / NT;
  dst[idx] = con[s] ? (gst ? gst[idx] : g ? g[s] : 0.0) : (src ? src[idx] : 0.0);
}
__global__ void k_axpy(int64_t n, double a, const double *__restrict__ x, double *__restrict__ y) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) y[i] = fma(a, x[i], y[i]);
}

NSTime make_nstime(const Temporal &T) {
  NSTime t{};
  for (int e = 0; e < T.nq * T.nq; ++e) {
    t.CE[e] = T.CE[e];
    t.Mt[e] = T.Mt[e];
  }
  for (int e = 0; e < T.nq * T.nq * T.nq; ++e) t.T[e] = T.T[e];
  return t;
}

template <class F>
void by_nq(int nq, F f) {
  switch (nq) {
    case 1: f(std::integral_constant<int, 1>()); break;
    case 2: f(std::integral_constant<int, 2>()); break;
    case 3: f(std::integral_constant<int, 3>()); break;
    default: f(std::integral_constant<int, 4>()); break;
  }
}

}  // namespace

void launch_ns_mask(int64_t ns, int64_t NT, const uint8_t *con, const double *g, const double *src, double *dst,
                    cudaStream_t s, const double *gst) {
  const int64_t n = ns * NT;
  k_ns_mask<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(ns, NT, con, g, gst, src, dst);
  ++g_launches;
}

void launch_axpy(int64_t n, double a, const double *x, double *y, cudaStream_t s) {
  k_axpy<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(n, a, x, y);
  ++g_launches;
}

size_t ns_factor_smem(int m, int mp) {
  return ((size_t)m * m + ns_factor_xdoubles(m)) * sizeof(double) + (size_t)(2 * m + mp) * sizeof(int) + 16;
}

size_t ns_sweep_smem(int m, int mp, int64_t mstride, bool staged) {
  return ((staged ? 2 * mstride : 0) + (int64_t)mp * mp + 2 * m + 2 * mp + 256) * sizeof(double) + mp * sizeof(int) +
         16;
}

void launch_ns_assemble_linear(const NSGeom &g, const DevCSR &A, const double *ref, cudaStream_t s) {
  k_ns_assemble_linear<<<(unsigned)((g.ns + 127) / 128), 128, 0, s>>>(g, A.rowptr, A.col, A.val, A.val2, ref);
  ++g_launches;
}

void launch_ns_assemble_conv(const NSGeom &g, int64_t NT, double R, bool newton, const DevCSR &A, const int32_t *vvptr,
                             const double *W, double *conv, const double *Th, cudaStream_t s) {
  const size_t sm = (size_t)2 * g.nu * g.nu * g.nu * sizeof(double);
  const int64_t n = g.Lu * NT;
  k_ns_assemble_conv<<<(unsigned)((n + 255) / 256), 256, sm, s>>>(g, NT, R, newton ? 1 : 0, A.rowptr, A.col, vvptr, W,
                                                                  conv, Th);
  ++g_launches;
}

void launch_ns_inject(const NSGeom &c, const NSGeom &f, int64_t NT, const double *Wf, double *Wc, cudaStream_t s,
                      const NSInjMap *map) {
  NSInjMap m{0, 0, 0, f.Lux - 1, 0, f.Lpx - 1};
  if (map) m = *map;
  const int64_t n = c.ns * NT;
  k_ns_inject<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(c, f, NT, Wf, Wc, m);
  ++g_launches;
}

void launch_ns_residual(const NSGeom &g, int q, int N, const Temporal &T, const DevCSR &A, const int32_t *vvptr,
                        const double *conv, const uint8_t *con, const double *u, const double *b, double *r,
                        cudaStream_t s) {
  const NSTime tm = make_nstime(T);
  const unsigned blocks = (unsigned)((g.ns + 7) / 8);
  by_nq(q + 1, [&](auto NQc) {
    constexpr int NQ = decltype(NQc)::value;
    k_ns_residual<NQ><<<blocks, 256, 0, s>>>(g.ns, N, A.rowptr, A.col, A.val, A.val2, 2 * g.Lu, vvptr, conv, con, u,
                                             b, r, tm);
  });
  ++g_launches;
}

void launch_ns_patch_pos(const NSGeom &g, const DevCSR &A, const int32_t *vvptr, const int32_t *pnodes, int64_t npatch,
                         int mp, int32_t *ppos, int32_t *pvv, cudaStream_t s) {
  if (npatch <= 0) return;
  k_ns_patch_pos<<<(unsigned)npatch, 256, 0, s>>>(mp, pnodes, A.rowptr, A.col, 2 * g.Lu, vvptr, ppos, pvv);
  ++g_launches;
}

void launch_ns_factor(const NSGeom &g, int q, int N, const Temporal &T, const DevCSR &A, const int32_t *vvptr,
                      const double *conv, const int32_t *pnodes, int64_t npatch, int mp, int64_t mstride, double *out,
                      int32_t *info, const int32_t *ppos, const int32_t *pvv, cudaStream_t s,
                      int n0, int nwin) {
  const NSTime tm = make_nstime(T);
  const int m = (q + 1) * mp;
  if (nwin <= 0) nwin = N;  // slab window [n0, n0 + nwin): out holds npatch x nwin inverses
  const size_t sm = ns_factor_smem(m, mp);
  const size_t sml = sm + (size_t)2 * m * sizeof(int) + (size_t)m + 8;  // + rowmap, tmp, used_in
  dim3 grid((unsigned)npatch, (unsigned)nwin);
  // row-per-thread register Gauss-Jordan, fully unrolled (instantiated for DG0 / DG1 patch sizes only:
  // each instance is ~7k straight-line DFMAs)
  // The shared-memory blocked kernel (gj_invert_smem: DMMA tile updates, 2.5 TF/s at
  // m = 78) is the default for every m; WRMG_NS_FACTOR_REG=1 selects the register
  // Gauss-Jordan kernels below for m <= 80 (1.9 TF/s at m = 78; A/B).
  static const bool force_smem = [] {
    const char *e = getenv("WRMG_NS_FACTOR_REG");
    return !(e && e[0] == '1');
  }();
  if (!force_smem && nwin == N && q == 0 && m <= 64) {
    k_ns_factor_row<1, 64, 64><<<grid, 64, 0, s>>>(mp, N, mstride, pnodes, A.val, A.val2, conv, tm, out, info, ppos,
                                                   pvv);
    ++g_launches;
    return;
  }
  if (!force_smem && nwin == N && q == 1 && m <= 80) {
    k_ns_factor_row<2, 80, 96><<<grid, 96, 0, s>>>(mp, N, mstride, pnodes, A.val, A.val2, conv, tm, out, info, ppos,
                                                   pvv);
    ++g_launches;
    return;
  }
  if (!force_smem && nwin == N && m <= 80) {  // register-tiled Gauss-Jordan (4 x 8 tiles, 20 x 10 threads)
    by_nq(q + 1, [&](auto NQc) {
      constexpr int NQ = decltype(NQc)::value;
      k_ns_factor_reg<NQ, 4, 8, 20, 10><<<grid, 256, 0, s>>>(mp, N, mstride, pnodes, A.val, A.val2, conv, tm, out,
                                                             info, ppos, pvv);
    });
    ++g_launches;
    return;
  }
  // warp-panel Gauss-Jordan (gj_invert_smem_wp) for m <= 192; WRMG_NS_FACTOR_WP=0: the
  // column-at-a-time panels of gj_invert_smem (A/B)
  static const bool wp = [] {
    const char *e = getenv("WRMG_NS_FACTOR_WP");
    return !(e && e[0] == '0');
  }();
  // look-ahead panels without row interchanges (gj_invert_smem_lr, default); WRMG_NS_FACTOR_LA=1:
  // look-ahead with interchanges (gj_invert_smem_la), 0: neither (A/B)
  static const int la = [] {
    const char *e = getenv("WRMG_NS_FACTOR_LA");
    return e ? (e[0] == '0' ? 0 : e[0] == '1' ? 1 : 2) : 2;
  }();
  // register-tiled Gauss-Jordan (k_ns_factor_rt) for the Vanka block sizes m <= 96 of the
  // Taylor-Hood levels (P2-P1: m = 39 (DG0), 78 (DG1); P3-P2: m = 81 (DG0));
  // WRMG_NS_FACTOR_RT=0 selects the shared-memory kernels below (A/B), =9 the phase-timer
  // build read by tools/rt_prof.py
  static const int rt = [] {
    const char *e = getenv("WRMG_NS_FACTOR_RT");
    return e ? e[0] - '0' : 1;
  }();
  if (rt && force_smem) {
    auto go = [&](auto kern, int nt) {
      const int thr = 32 * ((nt + 1) / 2 + 1);
      static const size_t pad = [] {  // experiments: WRMG_RT_SMEM_PAD=<KB> lowers the CTAs per SM
        const char *e = getenv("WRMG_RT_SMEM_PAD");
        return e ? (size_t)atoi(e) * 1024 : 0;
      }();
      const size_t smr = pad + std::max(ns_factor_rt_smem<5>(m, mp), std::max(ns_factor_rt_smem<10>(m, mp),
                                                                             ns_factor_rt_smem<11>(m, mp)));
      smem_optin((const void *)kern, (int)smr);
      kern<<<grid, thr, smr, s>>>(mp, N, mstride, pnodes, A.val, A.val2, conv, tm, out, info, ppos, pvv, n0, nwin);
      ++g_launches;
    };
    const int nt = (m + 7) / 8;
    if (q == 0 && nt == 5) return go(k_ns_factor_rt<1, 5, 3>, 5);
    if (q == 1 && nt == 10 && rt == 9) return go(k_ns_factor_rt<2, 10, 3, true>, 10);
    if (q == 1 && nt == 10) return go(k_ns_factor_rt<2, 10, 3>, 10);
    if (q == 0 && nt == 11) return go(k_ns_factor_rt<1, 11, 2>, 11);
  }
  by_nq(q + 1, [&](auto NQc) {
    constexpr int NQ = decltype(NQc)::value;
    // WRMG_NS_FACTOR_WARP=1: one warp per block, four blocks per CTA (measured slower:
    // C3 factor@L4 134 vs 86 ms -- one warp per scheduler exposes every latency)
    static const bool warp_blocks = [] {
      const char *e = getenv("WRMG_NS_FACTOR_WARP");
      return e && e[0] == '1';
    }();
    const size_t perw = ns_factor_warp_doubles(m, mp) * sizeof(double);
    if (warp_blocks && nwin == N && wp && m <= 96 && perw <= 56 * 1024) {
      const int wpb = (int)std::min<size_t>(4, (220 * 1024) / perw);
      const int64_t nblk = npatch * N;
      const int grid = (int)std::min<int64_t>((nblk + wpb - 1) / wpb, (int64_t)8 * num_sms());
      const size_t smw = perw * wpb;
      if (wpb == 4) {
        smem_optin((const void *)k_ns_factor_warp<NQ, 4, 3>, (int)smw);
        k_ns_factor_warp<NQ, 4, 3><<<grid, 128, smw, s>>>(mp, N, nblk, mstride, pnodes, A.val, A.val2, conv, tm, out,
                                                          info, ppos, pvv);
      } else {
        smem_optin((const void *)k_ns_factor_warp<NQ, 1, 3>, (int)perw);
        k_ns_factor_warp<NQ, 1, 3><<<grid, 32, perw, s>>>(mp, N, nblk, mstride, pnodes, A.val, A.val2, conv, tm, out,
                                                         info, ppos, pvv);
      }
    } else if (wp && la == 2 && m <= 96) {
      smem_optin((const void *)k_ns_factor<NQ, 128, 3, 2>, (int)sml);
      k_ns_factor<NQ, 128, 3, 2><<<grid, 128, sml, s>>>(mp, N, mstride, pnodes, A.rowptr, A.col, A.val, A.val2,
                                                        2 * g.Lu, vvptr, conv, tm, out, info, ppos, pvv, n0, nwin);
    } else if (wp && la == 2 && m <= 192) {
      smem_optin((const void *)k_ns_factor<NQ, 256, 6, 2>, (int)sml);
      k_ns_factor<NQ, 256, 6, 2><<<grid, 256, sml, s>>>(mp, N, mstride, pnodes, A.rowptr, A.col, A.val, A.val2,
                                                        2 * g.Lu, vvptr, conv, tm, out, info, ppos, pvv, n0, nwin);
    } else if (wp && la == 1 && m <= 96) {
      smem_optin((const void *)k_ns_factor<NQ, 128, 3, 1>, (int)sm);
      k_ns_factor<NQ, 128, 3, 1><<<grid, 128, sm, s>>>(mp, N, mstride, pnodes, A.rowptr, A.col, A.val, A.val2,
                                                       2 * g.Lu, vvptr, conv, tm, out, info, ppos, pvv, n0, nwin);
    } else if (wp && la == 1 && m <= 192) {
      smem_optin((const void *)k_ns_factor<NQ, 256, 6, 1>, (int)sm);
      k_ns_factor<NQ, 256, 6, 1><<<grid, 256, sm, s>>>(mp, N, mstride, pnodes, A.rowptr, A.col, A.val, A.val2,
                                                       2 * g.Lu, vvptr, conv, tm, out, info, ppos, pvv, n0, nwin);
    } else if (wp && m <= 96) {
      smem_optin((const void *)k_ns_factor<NQ, 128, 3>, (int)sm);
      k_ns_factor<NQ, 128, 3><<<grid, 128, sm, s>>>(mp, N, mstride, pnodes, A.rowptr, A.col, A.val, A.val2, 2 * g.Lu,
                                                    vvptr, conv, tm, out, info, ppos, pvv, n0, nwin);
    } else if (wp && m <= 192) {
      smem_optin((const void *)k_ns_factor<NQ, 256, 6>, (int)sm);
      k_ns_factor<NQ, 256, 6><<<grid, 256, sm, s>>>(mp, N, mstride, pnodes, A.rowptr, A.col, A.val, A.val2, 2 * g.Lu,
                                                    vvptr, conv, tm, out, info, ppos, pvv, n0, nwin);
    } else {
      smem_optin((const void *)k_ns_factor<NQ, 256, 0>, (int)sm);
      k_ns_factor<NQ, 256, 0><<<grid, 256, sm, s>>>(mp, N, mstride, pnodes, A.rowptr, A.col, A.val, A.val2, 2 * g.Lu,
                                                    vvptr, conv, tm, out, info, ppos, pvv, n0, nwin);
    }
  });
  ++g_launches;
}

void launch_ns_sweep(int q, int N, int mp, int64_t npatch, int64_t mstride, const int32_t *pnodes, const double *wnode,
                     const DevCSR &A, const double *Dinv, const double *r, double *u, double omega, cudaStream_t s,
                     int n0, int nwin, double *xs) {
  const int m = (q + 1) * mp;
  if (nwin <= 0) nwin = N;
  // m <= 256 (one thread per patch row) is enforced by setup_ns
  const bool staged = ns_sweep_smem(m, mp, mstride, true) <= 200 * 1024;
  const size_t sm = ns_sweep_smem(m, mp, mstride, staged);
  if (!staged) {  // chunked ring: two CTAs per SM when it fits, else one with a deeper ring
    const size_t fixed = ((size_t)mp * mp + 2 * m + mp) * sizeof(double) + mp * sizeof(int) + 64;
    int CW = 16, R = 2;
    while (CW > 4 && fixed + (size_t)R * CW * m * sizeof(double) > 110 * 1024) CW /= 2;
    if (fixed + (size_t)R * CW * m * sizeof(double) > 110 * 1024) {
      CW = 32;
      R = 3;
      while (CW > 4 && fixed + (size_t)R * CW * m * sizeof(double) > 220 * 1024) CW /= 2;
    }
    const size_t smc = fixed + (size_t)R * CW * m * sizeof(double);
    by_nq(q + 1, [&](auto NQc) {
      constexpr int NQ = decltype(NQc)::value;
      smem_optin((const void *)k_ns_sweep_chunked<NQ>, (int)smc);
      k_ns_sweep_chunked<NQ><<<(unsigned)npatch, 256, smc, s>>>(mp, N, mstride, CW, R, pnodes, wnode, A.rowptr,
                                                                A.col, A.val, Dinv, r, u, omega, n0, nwin,
                                                                xs);
    });
    ++g_launches;
    return;
  }
  by_nq(q + 1, [&](auto NQc) {
    constexpr int NQ = decltype(NQc)::value;
    if (staged) {
      smem_optin((const void *)k_ns_sweep<NQ, true>, (int)sm);
      k_ns_sweep<NQ, true><<<(unsigned)npatch, 256, sm, s>>>(mp, N, mstride, pnodes, wnode, A.rowptr, A.col, A.val,
                                                             Dinv, r, u, omega, n0, nwin, xs);
    } else {
      smem_optin((const void *)k_ns_sweep<NQ, false>, (int)sm);
      k_ns_sweep<NQ, false><<<(unsigned)npatch, 256, sm, s>>>(mp, N, mstride, pnodes, wnode, A.rowptr, A.col, A.val,
                                                              Dinv, r, u, omega, n0, nwin, xs);
    }
  });
  ++g_launches;
}

void launch_ns_project(double *P, int64_t nrow, int64_t NT, double *scratch, cudaStream_t s) {
  // scratch: >= (nb + 1) * NT doubles
  const int64_t rpb = std::max<int64_t>(16, (nrow + 295) / 296);
  const int nb = (int)((nrow + rpb - 1) / rpb);
  double *partial = scratch, *mean = scratch + (int64_t)nb * NT;
  k_colsum<<<nb, 256, 0, s>>>(P, nrow, NT, rpb, partial);
  k_colmean<<<(unsigned)((NT + 255) / 256), 256, 0, s>>>(partial, nb, NT, nrow, mean);
  const int64_t n = nrow * NT;
  k_colsub<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(P, nrow, NT, mean);
  g_launches += 3;
}

int64_t ns_project_scratch(int64_t nrow, int64_t NT) {
  const int64_t rpb = std::max<int64_t>(16, (nrow + 295) / 296);
  return ((nrow + rpb - 1) / rpb + 1) * NT;
}

void launch_ns_colsum_owned(const double *P, int Lx, int Ly, int c0, int nc, int64_t NT, double *scratch, double *sums,
                            cudaStream_t s) {
  // scratch: >= nb * NT doubles, nb = ceil(Ly / rpb); sums: NT doubles
  const int rpb = std::max(1, (Ly + 295) / 296);
  const int nb = (Ly + rpb - 1) / rpb;
  k_colsum_cols<<<nb, 256, 0, s>>>(P, Lx, Ly, c0, nc, NT, rpb, scratch);
  k_colmean<<<(unsigned)((NT + 255) / 256), 256, 0, s>>>(scratch, nb, NT, 1, sums);
  g_launches += 2;
}

void launch_ns_sub_gathered_mean(double *P, int64_t nrow, int64_t NT, const double *gathered, int nranks,
                                 int64_t gnrow, double *mean, cudaStream_t s) {
  // mean = (sum over ranks, in rank order, of the owned column sums) / gnrow; P -= mean
  k_colmean<<<(unsigned)((NT + 255) / 256), 256, 0, s>>>(gathered, nranks, NT, gnrow, mean);
  const int64_t n = nrow * NT;
  k_colsub<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(P, nrow, NT, mean);
  g_launches += 2;
}

void launch_ns_coarse_blocks(const NSGeom &g, int q, int N, const Temporal &T, const DevCSR &A, const int32_t *vvptr,
                             const double *conv, const int32_t *cnodes, int mc, int pin, double *D, cudaStream_t s) {
  const NSTime tm = make_nstime(T);
  const int64_t m = (int64_t)(q + 1) * mc;
  dim3 grid((unsigned)std::min<int64_t>((m * m + 255) / 256, 1024), (unsigned)N);
  by_nq(q + 1, [&](auto NQc) {
    constexpr int NQ = decltype(NQc)::value;
    k_ns_coarse_blocks<NQ><<<grid, 256, 0, s>>>(mc, N, pin, cnodes, A.rowptr, A.col, A.val, A.val2, 2 * g.Lu, vvptr,
                                                conv, tm, D);
  });
  ++g_launches;
}

void launch_ns_coarse_H(int q, int N, int mc, int pin, const int32_t *cnodes, const int32_t *sid2c, const DevCSR &A,
                        const double *DinvT, double *H, double *G, cudaStream_t s) {
  const int m = (q + 1) * mc;
  dim3 grid((unsigned)((m + 127) / 128), (unsigned)mc, (unsigned)N);
  by_nq(q + 1, [&](auto NQc) {
    constexpr int NQ = decltype(NQc)::value;
    k_ns_coarse_H<NQ><<<grid, 128, 0, s>>>(mc, N, pin, cnodes, sid2c, A.rowptr, A.col, A.val, DinvT, H, G);
  });
  ++g_launches;
}

void launch_ns_coarse_solve_pint(int q, int N, int mc, int pin, const int32_t *cnodes, const double *DinvT,
                                 const double *H, const double *G, double *Zs, double *Ys, const double *r, double *z,
                                 int64_t ns, cudaStream_t s) {
  const int m = (q + 1) * mc;
  cudaMemsetAsync(z, 0, ns * (int64_t)N * (q + 1) * sizeof(double), s);
  dim3 grid((unsigned)N, (unsigned)((m + 31) / 32));
  by_nq(q + 1, [&](auto NQc) {
    constexpr int NQ = decltype(NQc)::value;
    smem_optin((const void *)k_ns_coarse_pass<NQ, false>, m * (int)sizeof(double));
    smem_optin((const void *)k_ns_coarse_pass<NQ, true>, m * (int)sizeof(double));
    k_ns_coarse_pass<NQ, false><<<grid, 256, m * sizeof(double), s>>>(mc, N, pin, cnodes, DinvT, r, Zs, nullptr,
                                                                      nullptr, nullptr);
    if (10 * (size_t)mc * sizeof(double) <= 200 * 1024) {
      smem_optin((const void *)k_ns_coarse_yrec<NQ, 8>, 200 * 1024);
      k_ns_coarse_yrec<NQ, 8><<<1, 1024, 10 * mc * sizeof(double), s>>>(mc, N, Zs, G, Ys);
    } else {
      smem_optin((const void *)k_ns_coarse_yrec<NQ, 2>, 220 * 1024);
      k_ns_coarse_yrec<NQ, 2><<<1, 1024, 4 * mc * sizeof(double), s>>>(mc, N, Zs, G, Ys);
    }
    k_ns_coarse_pass<NQ, true><<<grid, 256, mc * sizeof(double), s>>>(mc, N, pin, cnodes, DinvT, r, Zs, H, Ys, z);
  });
  g_launches += 3;
}

void launch_ns_coarse_solve(int q, int N, int mc, int pin, const int32_t *cnodes, const DevCSR &A, const double *DinvT,
                            const double *r, double *z, double *xq, int64_t ns, int nnzj, cudaStream_t s) {
  const int m = (q + 1) * mc;
  cudaMemsetAsync(z, 0, ns * (int64_t)N * (q + 1) * sizeof(double), s);
  cudaMemsetAsync(xq, 0, ns * sizeof(double), s);
  const size_t sm = (m + 2 * ns + nnzj) * sizeof(double) + (nnzj + mc + 1) * sizeof(int);
  by_nq(q + 1, [&](auto NQc) {
    constexpr int NQ = decltype(NQc)::value;
    if (sm <= 200 * 1024 && m <= 512) {
      smem_optin((const void *)k_ns_coarse_cluster<NQ, 8>, (int)sm);
      k_ns_coarse_cluster<NQ, 8><<<8, 256, sm, s>>>(mc, N, pin, ns, cnodes, A.rowptr, A.col, A.val, DinvT, r, z,
                                                     nnzj);
    } else {
      k_ns_coarse_solve<NQ><<<1, 1024, m * sizeof(double), s>>>(mc, N, pin, cnodes, A.rowptr, A.col, A.val, DinvT, r,
                                                                z, xq);
    }
  });
  ++g_launches;
}

}  // namespace wrmg

// Tools only (not in include/wrmg.h): read and clear the k_ns_factor_rt phase timers
// (WRMG_NS_FACTOR_RT=9 builds them); out[16] = clock64 sums, out[15] = blocks.
extern "C" int wrmg_debug_rt_prof(unsigned long long *out) {
  if (cudaMemcpyFromSymbol(out, wrmg::g_rtprof, sizeof(unsigned long long) * 16) != cudaSuccess) return 1;
  unsigned long long z[16] = {0};
  return cudaMemcpyToSymbol(wrmg::g_rtprof, z, sizeof(z)) == cudaSuccess ? 0 : 1;
}
