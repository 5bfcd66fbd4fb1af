// Column kernels of the strip partition: halo pack / unpack (copy or add), ghost
// zeroing, and window copies between a rank's local lattice and the replicated
// global coarsest lattice.  A waveform-major vector v[(J Lx + I) NT + t] is
// viewed as (Ly, Lx, NT); a column block [c0, c0 + nc) is packed as (Ly, nc, NT).
#include <algorithm>

#include "internal.h"

namespace wrmg {
namespace {

// mode 0: buf = v[cols]; 1: v[cols] = buf; 2: v[cols] += buf; 3: v[cols] = 0
__global__ void k_cols(double *__restrict__ v, int Lx, int Ly, int64_t NT, int c0, int nc, double *__restrict__ buf,
                       int mode) {
  const int64_t n = (int64_t)Ly * nc * NT;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t t = e % NT, jc = e / NT;
    const int c = (int)(jc % nc), J = (int)(jc / nc);
    double *p = v + ((int64_t)J * Lx + c0 + c) * NT + t;
    switch (mode) {
      case 0: buf[e] = *p; break;
      case 1: *p = buf[e]; break;
      case 2: *p += buf[e]; break;
      default: *p = 0.0; break;
    }
  }
}

// dst[:, dc0 + c] = src[:, sc0 + c] for c < nc (lattices of widths Lxs / Lxd, same Ly)
__global__ void k_window(const double *__restrict__ src, int Lxs, int sc0, double *__restrict__ dst, int Lxd, int dc0,
                         int Ly, int nc, int64_t NT) {
  const int64_t n = (int64_t)Ly * nc * NT;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t t = e % NT, jc = e / NT;
    const int c = (int)(jc % nc), J = (int)(jc / nc);
    dst[((int64_t)J * Lxd + dc0 + c) * NT + t] = src[((int64_t)J * Lxs + sc0 + c) * NT + t];
  }
}

// out[e] = sum_q all[q n + e], q = 0 .. nchunks-1 in order (rank-order all-reduce:
// every rank forms bitwise-identical sums)
__global__ void k_sum_chunks(const double *__restrict__ all, int nchunks, int64_t n, double *__restrict__ out) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int q = 0; q < nchunks; ++q) s += all[(int64_t)q * n + e];
    out[e] = s;
  }
}

unsigned grid_for(int64_t n) { return (unsigned)std::min<int64_t>((n + 255) / 256, (int64_t)num_sms() * 16); }

}  // namespace

void launch_cols(double *v, int Lx, int Ly, int64_t NT, int c0, int nc, double *buf, int mode, cudaStream_t s) {
  if (nc <= 0) return;
  const int64_t n = (int64_t)Ly * nc * NT;
  k_cols<<<grid_for(n), 256, 0, s>>>(v, Lx, Ly, NT, c0, nc, buf, mode);
  ++g_launches;
}

void launch_window(const double *src, int Lxs, int sc0, double *dst, int Lxd, int dc0, int Ly, int nc, int64_t NT,
                   cudaStream_t s) {
  if (nc <= 0) return;
  const int64_t n = (int64_t)Ly * nc * NT;
  k_window<<<grid_for(n), 256, 0, s>>>(src, Lxs, sc0, dst, Lxd, dc0, Ly, nc, NT);
  ++g_launches;
}

void launch_sum_chunks(const double *all, int nchunks, int64_t n, double *out, cudaStream_t s) {
  k_sum_chunks<<<grid_for(n), 256, 0, s>>>(all, nchunks, n, out);
  ++g_launches;
}

}  // namespace wrmg
