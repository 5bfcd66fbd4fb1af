// Chebyshev-accelerated relaxation vector update and the
// initial-state right-hand side term (eq. dgintime, Y_0^- = y_0; R7).
#include <algorithm>

#include "internal.h"

namespace wrmg {
namespace {

// d = c1 d + c2 B r;  u += d   (three-term Chebyshev recurrence, DESIGN.md R-cheb)
__global__ void k_cheb_update(int64_t n, double c1, double c2, const double *__restrict__ br, double *__restrict__ d,
                              double *__restrict__ u) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double v = c1 != 0.0 ? fma(c1, d[i], c2 * br[i]) : c2 * br[i];  // first step: d not read
    d[i] = v;
    u[i] += v;
  }
}

// b[i, slab 0, a] += phi_a(0) (M u0)_i on free rows (thread per lattice node)
struct Phi0 {
  double v[4];
};
__global__ void k_rhs_initial(int64_t nnode, int nq, int64_t NT, Phi0 phi, const int32_t *__restrict__ rowptr,
                              const int32_t *__restrict__ col, const double *__restrict__ Mv,
                              const uint8_t *__restrict__ con, const double *__restrict__ u0, double *__restrict__ b) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= nnode || con[i]) return;
  double s = 0.0;
  for (int e = rowptr[i]; e < rowptr[i + 1]; ++e) s = fma(Mv[e], u0[col[e]], s);
  for (int a = 0; a < nq; ++a) b[i * NT + a] += phi.v[a] * s;
}

}  // namespace

void launch_cheb_update(int64_t n, double c1, double c2, const double *br, double *d, double *u, cudaStream_t s) {
  const unsigned grid = (unsigned)std::min<int64_t>((n + 255) / 256, (int64_t)num_sms() * 16);
  k_cheb_update<<<grid, 256, 0, s>>>(n, c1, c2, br, d, u);
  ++g_launches;
}

void launch_rhs_initial(const Level &L, int nq, int64_t NT, const double *phi0, const double *u0, double *b,
                        cudaStream_t s) {
  Phi0 p{};
  for (int a = 0; a < nq; ++a) p.v[a] = phi0[a];
  k_rhs_initial<<<(unsigned)((L.nnode + 127) / 128), 128, 0, s>>>(L.nnode, nq, NT, p, L.A.rowptr, L.A.col, L.A.val,
                                                                   L.con, u0, b);
  ++g_launches;
}

}  // namespace wrmg
