// FGMRES building blocks (H13), fused so that one Arnoldi step of classical
// Gram-Schmidt applied twice (CGS2, R16) streams the basis three times instead
// of four:
//   pass A:  h  = V^T w
//   pass B:  w <- w - V h,   h2 = V^T w        (one read of V and w, one write of w)
//   pass C:  w <- w - V h2,  |w|^2
// Every kernel uses a fixed grid and a fixed two-stage reduction order, so dot
// products are bitwise reproducible run to run.
#include "internal.h"

namespace wrmg {
namespace {

constexpr int kMaxV = 32;

struct Ptrs {
  const double *p[kMaxV];
};

// MODE 0: part[k] = sum_i V_k[i] w[i]
// MODE 1: w <- w - sum_k c_k V_k;  part[k] = sum_i V_k[i] w_new[i]
// MODE 2: w <- w - sum_k c_k V_k;  part[0] = sum_i w_new[i]^2
// MODE 3: w <- w + sgn sum_k c_k V_k  (MODEs 1, 2 subtract: sgn = -1)
template <int NV, int MODE, bool VEC = true>
__global__ void __launch_bounds__(256) k_krylov(Ptrs V, int nv, double *__restrict__ w, const double *__restrict__ coef,
                                                int64_t n, double *__restrict__ partials, int stride, double sgn) {
  double acc[NV];
  double c[NV];
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    acc[k] = 0.0;
    c[k] = (MODE != 0 && k < nv) ? sgn * coef[k] : 0.0;
  }
  // element i (scalar tail) or the pair (2 i, 2 i + 1) of 16-byte loads: twice the bytes in
  // flight per thread of the scalar form (the early Arnoldi steps stream only 1-3 vectors)
  // VEC = false (a vector not 16-byte aligned): one element per iteration
  const int64_t n2 = VEC ? n >> 1 : 0;
  const int64_t gstride = (int64_t)gridDim.x * blockDim.x;
  const int64_t nit = VEC ? n2 + (n & 1) : n;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nit; i += gstride) {
    const bool pair = VEC && i < n2;
    const int64_t is = VEC ? 2 * i : i;  // the scalar element
    double2 wv = pair ? reinterpret_cast<const double2 *>(w)[i] : make_double2(w[is], 0.0);
    if (MODE != 0) {
      double2 v[NV];
#pragma unroll
      for (int k = 0; k < NV; ++k)
        v[k] = k < nv ? (pair ? __ldg(reinterpret_cast<const double2 *>(V.p[k]) + i)
                              : make_double2(__ldg(V.p[k] + is), 0.0))
                      : make_double2(0.0, 0.0);
      double2 sv = wv;
#pragma unroll
      for (int k = 0; k < NV; ++k) {
        sv.x = fma(c[k], v[k].x, sv.x);
        sv.y = fma(c[k], v[k].y, sv.y);
      }
      wv = sv;
      if (pair) reinterpret_cast<double2 *>(w)[i] = wv;
      else w[is] = wv.x;
      if (MODE == 1) {
#pragma unroll
        for (int k = 0; k < NV; ++k) acc[k] = fma(v[k].y, wv.y, fma(v[k].x, wv.x, acc[k]));
      } else if (MODE == 2) {
        acc[0] = fma(wv.y, wv.y, fma(wv.x, wv.x, acc[0]));
      }
    } else {
#pragma unroll
      for (int k = 0; k < NV; ++k)
        if (k < nv) {
          const double2 vk = pair ? __ldg(reinterpret_cast<const double2 *>(V.p[k]) + i)
                                  : make_double2(__ldg(V.p[k] + is), 0.0);
          acc[k] = fma(vk.y, wv.y, fma(vk.x, wv.x, acc[k]));
        }
    }
  }
  if (MODE == 3) return;
  constexpr int NR = (MODE == 2) ? 1 : NV;
  __shared__ double red[8][NR];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < NR; ++k) {
    double v = acc[k];
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) red[wid][k] = v;
  }
  __syncthreads();
  const int nout = (MODE == 2) ? 1 : nv;
  if (threadIdx.x < nout) {
    double s = 0.0;
    for (int k = 0; k < 8; ++k) s += red[k][threadIdx.x];
    partials[(int64_t)blockIdx.x * stride + threadIdx.x] = s;
  }
}

__global__ void k_reduce(const double *__restrict__ partials, int nblk, int nv, double *__restrict__ out) {
  const int v = blockIdx.x;
  const int lane = threadIdx.x;
  double s = 0.0;
  for (int b = lane; b < nblk; b += 32) s += partials[(int64_t)b * nv + v];
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) out[v] = s;
}

// Device-side CGS2 coefficients of FGMRES step j with the lazily scaled basis (single
// rank: no host round trip inside the Arnoldi step).  kry layout (doubles):
//   [0, 32) sc_i   [32, 64) h_i = <V_i', w'>   [64, 96) sc_i^2 h_i   [96, 128) h2_i
//   [128, 160) sc_i^2 h2_i   [160, 192) Hessenberg column   [192] |w'|^2   [200, 233) out
// stage 0 (after pass A): coef A, column = sc_i sc_j h_i; stage 1 (after pass B): coef B,
// column += sc_i sc_j h2_i; stage 2 (after pass C): sc_{j+1} = 1 / |w'|, out = (column, |w'|^2).
// The products are rounded one at a time (__dmul_rn), as the host computes them.
__global__ void k_cgs_step(double *__restrict__ kry, int j, int stage) {
  const int i = threadIdx.x;
  double *sc = kry, *h = kry + 32, *ca = kry + 64, *h2 = kry + 96, *cb = kry + 128, *col = kry + 160;
  if (stage == 0 && i <= j) {
    ca[i] = __dmul_rn(__dmul_rn(sc[i], sc[i]), h[i]);
    col[i] = __dmul_rn(__dmul_rn(sc[i], sc[j]), h[i]);
  } else if (stage == 1 && i <= j) {
    cb[i] = __dmul_rn(__dmul_rn(sc[i], sc[i]), h2[i]);
    col[i] = __dadd_rn(col[i], __dmul_rn(__dmul_rn(sc[i], sc[j]), h2[i]));
  } else if (stage == 2) {
    if (i <= j) kry[200 + i] = col[i];
    if (i == 0) {
      kry[200 + j + 1] = kry[192];
      if (j + 1 < 32) sc[j + 1] = 1.0 / sqrt(kry[192]);
    }
  }
}

__global__ void k_scale(double *__restrict__ dst, const double *__restrict__ src, double a, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = a * src[i];
}

int grid_for(int64_t n) { return (int)std::min<int64_t>((n + 255) / 256, (int64_t)num_sms() * 8); }

template <int MODE>
void krylov_launch(const double *const *V, int nv, double *w, const double *coef, int64_t n, double *partials,
                   int nblk, cudaStream_t s, double sgn = -1.0) {
  Ptrs P{};
  uintptr_t al = (uintptr_t)w;
  for (int k = 0; k < nv; ++k) {
    P.p[k] = V[k];
    al |= (uintptr_t)V[k];
  }
  const int stride = (MODE == 2) ? 1 : nv;
  if (al & 15) {  // a vector not 16-byte aligned (e.g. a user's tensor view): the scalar form
    k_krylov<32, MODE, false><<<nblk, 256, 0, s>>>(P, nv, w, coef, n, partials, stride, sgn);
    ++g_launches;
    return;
  }
  if (nv <= 4) k_krylov<4, MODE><<<nblk, 256, 0, s>>>(P, nv, w, coef, n, partials, stride, sgn);
  else if (nv <= 8) k_krylov<8, MODE><<<nblk, 256, 0, s>>>(P, nv, w, coef, n, partials, stride, sgn);
  else if (nv <= 16) k_krylov<16, MODE><<<nblk, 256, 0, s>>>(P, nv, w, coef, n, partials, stride, sgn);
  else k_krylov<32, MODE><<<nblk, 256, 0, s>>>(P, nv, w, coef, n, partials, stride, sgn);
  ++g_launches;
}

}  // namespace

int multidot_blocks(int64_t n) { return (int)std::min<int64_t>(std::min(4 * num_sms(), kDotBlocksMax), (n + 255) / 256); }

void launch_multidot(const double *const *V, int nv, const double *w, int64_t n, double *partials, int nblk,
                     cudaStream_t s) {
  krylov_launch<0>(V, nv, const_cast<double *>(w), nullptr, n, partials, nblk, s);
}

void launch_cgs_update_dot(const double *const *V, int nv, double *w, const double *coef, int64_t n,
                           double *partials, int nblk, cudaStream_t s) {
  krylov_launch<1>(V, nv, w, coef, n, partials, nblk, s);
}

void launch_cgs_update_norm(const double *const *V, int nv, double *w, const double *coef, int64_t n,
                            double *partials, int nblk, cudaStream_t s) {
  krylov_launch<2>(V, nv, w, coef, n, partials, nblk, s);
}

void launch_reduce_partials(const double *partials, int nblk, int nv, double *out, cudaStream_t s) {
  k_reduce<<<nv, 32, 0, s>>>(partials, nblk, nv, out);
  ++g_launches;
}

void launch_multiaxpy(double *w, const double *const *V, const double *coef_dev, int nv, int64_t n, double sign,
                      cudaStream_t s) {
  // sign +1: w += V c (solution update); sign -1: w -= V c
  krylov_launch<3>(V, nv, w, coef_dev, n, nullptr, grid_for(n), s, sign);
}

void launch_cgs_step(double *kry, int j, int stage, cudaStream_t s) {
  k_cgs_step<<<1, 32, 0, s>>>(kry, j, stage);
  ++g_launches;
}

void launch_scale(double *dst, const double *src, double a, int64_t n, cudaStream_t s) {
  k_scale<<<grid_for(n), 256, 0, s>>>(dst, src, a, n);
  ++g_launches;
}

}  // namespace wrmg
