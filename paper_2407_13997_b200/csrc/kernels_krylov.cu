// FGMRES building blocks (H13): fused multi-vector dot products (one pass over
// w for up to 8 basis vectors), deterministic two-stage reduction, fused
// multi-AXPY, scaling.  Fixed grid and fixed reduction order -> bitwise
// reproducible dots.
#include "internal.h"

namespace wrmg {
namespace {

constexpr int kDotBlocks = 148 * 4;
constexpr int kGroup = 8;

struct Ptrs {
  const double *p[kGroup];
};

template <int G>
__global__ void __launch_bounds__(256) k_multidot(Ptrs V, const double *__restrict__ w, int64_t n,
                                                  double *__restrict__ partials, int stride, int v0) {
  double acc[G];
#pragma unroll
  for (int g = 0; g < G; ++g) acc[g] = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double wv = __ldg(w + i);
#pragma unroll
    for (int g = 0; g < G; ++g) acc[g] = fma(__ldg(V.p[g] + i), wv, acc[g]);
  }
  __shared__ double red[8][G];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int g = 0; g < G; ++g) {
    double v = acc[g];
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) red[wid][g] = v;
  }
  __syncthreads();
  if (threadIdx.x < G) {
    double s = 0.0;
    for (int k = 0; k < 8; ++k) s += red[k][threadIdx.x];
    partials[(int64_t)blockIdx.x * stride + v0 + threadIdx.x] = s;
  }
}

__global__ void k_reduce(const double *__restrict__ partials, int nblk, int nv, double *__restrict__ out) {
  // one warp per output value, fixed order
  const int v = blockIdx.x;
  const int lane = threadIdx.x;
  double s = 0.0;
  for (int b = lane; b < nblk; b += 32) s += partials[(int64_t)b * nv + v];
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) out[v] = s;
}

template <int G>
__global__ void __launch_bounds__(256) k_multiaxpy(double *__restrict__ w, Ptrs V, const double *__restrict__ coef,
                                                   int64_t n, double sign) {
  double c[G];
#pragma unroll
  for (int g = 0; g < G; ++g) c[g] = sign * coef[g];
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double acc = w[i];
#pragma unroll
    for (int g = 0; g < G; ++g) acc = fma(c[g], __ldg(V.p[g] + i), acc);
    w[i] = acc;
  }
}

__global__ void k_scale(double *__restrict__ dst, const double *__restrict__ src, double a, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = a * src[i];
}

int grid_for(int64_t n) { return (int)std::min<int64_t>((n + 255) / 256, 148 * 8); }

}  // namespace

int multidot_blocks(int64_t n) { return (int)std::min<int64_t>(kDotBlocks, (n + 255) / 256); }

void launch_multidot(const double *const *V, int nv, const double *w, int64_t n, double *partials, int nblk,
                     cudaStream_t s) {
  for (int v0 = 0; v0 < nv; v0 += kGroup) {
    Ptrs P{};
    int G = std::min(kGroup, nv - v0);
    for (int g = 0; g < G; ++g) P.p[g] = V[v0 + g];
    switch (G) {
#define C(GG) case GG: k_multidot<GG><<<nblk, 256, 0, s>>>(P, w, n, partials, nv, v0); ++g_launches; break;
      C(1) C(2) C(3) C(4) C(5) C(6) C(7) C(8)
#undef C
    }
  }
}

void launch_reduce_partials(const double *partials, int nblk, int nv, double *out, cudaStream_t s) {
  k_reduce<<<nv, 32, 0, s>>>(partials, nblk, nv, out); ++g_launches;
}

void launch_multiaxpy(double *w, const double *const *V, const double *coef_dev, int nv, int64_t n, double sign,
                      cudaStream_t s) {
  for (int v0 = 0; v0 < nv; v0 += kGroup) {
    Ptrs P{};
    int G = std::min(kGroup, nv - v0);
    for (int g = 0; g < G; ++g) P.p[g] = V[v0 + g];
    switch (G) {
#define C(GG) case GG: k_multiaxpy<GG><<<grid_for(n), 256, 0, s>>>(w, P, coef_dev + v0, n, sign); ++g_launches; break;
      C(1) C(2) C(3) C(4) C(5) C(6) C(7) C(8)
#undef C
    }
  }
}

void launch_scale(double *dst, const double *src, double a, int64_t n, cudaStream_t s) {
  k_scale<<<grid_for(n), 256, 0, s>>>(dst, src, a, n); ++g_launches;
}

}  // namespace wrmg
