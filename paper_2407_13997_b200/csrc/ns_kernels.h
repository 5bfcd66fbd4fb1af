// Launchers of the Navier-Stokes kernels (kernels_ns.cu).
#pragma once
#include <type_traits>

#include "internal.h"
#include "ns.h"

namespace wrmg {

// Geometry of one Taylor-Hood level, passed by value to kernels.
struct NSGeom {
  int nx, ny, ku, kp, Lux, Lpx, nu, np;
  int64_t Lu, Lp, ns;
  double h;
};

struct NSTime {
  double CE[16], Mt[16], T[64];
};

size_t ns_factor_smem(int m, int mp);
size_t ns_sweep_smem(int m, int mp, int64_t mstride, bool staged);
int64_t ns_project_scratch(int64_t nrow, int64_t NT);

void launch_ns_assemble_linear(const NSGeom &g, const DevCSR &A, const double *ref, cudaStream_t s);
void launch_ns_assemble_conv(const NSGeom &g, int64_t NT, double R, bool newton, const DevCSR &A, const int32_t *vvptr,
                             const double *W, double *conv, const double *Th, cudaStream_t s);
// Injection fine -> coarse (R13): coarse local column I reads fine local column 2 I + du
// (velocity) / 2 I + dp (pressure); outside [fu0, fu1] / [fp0, fp1] the coarse value is 0
// (strips: only the owned fine columns are read; the rest is refreshed from the owners).
struct NSInjMap {
  int du, dp, fu0, fu1, fp0, fp1;
};
void launch_ns_inject(const NSGeom &c, const NSGeom &f, int64_t NT, const double *Wf, double *Wc, cudaStream_t s,
                      const NSInjMap *map = nullptr);
void launch_ns_residual(const NSGeom &g, int q, int N, const Temporal &T, const DevCSR &A, const int32_t *vvptr,
                        const double *conv, const uint8_t *con, const double *u, const double *b, double *r,
                        cudaStream_t s);
void launch_ns_factor(const NSGeom &g, int q, int N, const Temporal &T, const DevCSR &A, const int32_t *vvptr,
                      const double *conv, const int32_t *pnodes, int64_t npatch, int mp, int64_t mstride, double *out,
                      int32_t *info, const int32_t *ppos, const int32_t *pvv, cudaStream_t s, int n0 = 0,
                      int nwin = 0);
void launch_ns_patch_pos(const NSGeom &g, const DevCSR &A, const int32_t *vvptr, const int32_t *pnodes, int64_t npatch,
                         int mp, int32_t *ppos, int32_t *pvv, cudaStream_t s);
void launch_ns_sweep(int q, int N, int mp, int64_t npatch, int64_t mstride, const int32_t *pnodes, const double *wnode,
                     const DevCSR &A, const double *Dinv, const double *r, double *u, double omega, cudaStream_t s,
                     int n0 = 0, int nwin = 0, double *xs = nullptr);
void launch_ns_project(double *P, int64_t nrow, int64_t NT, double *scratch, cudaStream_t s);
// Strip form of the projection: column sums over the owned lattice columns (scratch >=
// (Ly + 1) NT), then, from the all-gathered per-rank sums, P -= sum / gnrow.
void launch_ns_colsum_owned(const double *P, int Lx, int Ly, int c0, int nc, int64_t NT, double *scratch, double *sums,
                            cudaStream_t s);
void launch_ns_sub_gathered_mean(double *P, int64_t nrow, int64_t NT, const double *gathered, int nranks,
                                 int64_t gnrow, double *mean, cudaStream_t s);
void launch_ns_coarse_blocks(const NSGeom &g, int q, int N, const Temporal &T, const DevCSR &A, const int32_t *vvptr,
                             const double *conv, const int32_t *cnodes, int mc, int pin, double *D, cudaStream_t s);
void launch_ns_coarse_solve(int q, int N, int mc, int pin, const int32_t *cnodes, const DevCSR &A, const double *DinvT,
                            const double *r, double *z, double *xq, int64_t ns, int nnzj, cudaStream_t s);
void launch_ns_mask(int64_t ns, int64_t NT, const uint8_t *con, const double *g, const double *src, double *dst,
                    cudaStream_t s, const double *gst = nullptr);
void launch_axpy(int64_t n, double a, const double *x, double *y, cudaStream_t s);
// Batched inverse from LU factors (kernels_setup.cu): out[b] = column-major inverse of batch b.
// Blocked Gauss-Jordan inverses (kernels_gj.cu) for large blocks: A (batch
// column-major m x m, destroyed), piv (batch x m), info (batch: 0 or 1 + first
// singular column), out (batch column-major inverses), scratch of
// gj_scratch_doubles(m, batch) doubles.
constexpr int kGJMinM = 192;  // below this the CTA-per-matrix LU + inverse is used
size_t gj_scratch_doubles(int m, int batch);
void launch_gj_inverse_batched(double *A, int m, int batch, int32_t *piv, int32_t *info, double *out,
                               double *scratch, cudaStream_t s);
void launch_ns_coarse_H(int q, int N, int mc, int pin, const int32_t *cnodes, const int32_t *sid2c, const DevCSR &A,
                        const double *DinvT, double *H, double *G, cudaStream_t s);
void launch_ns_coarse_solve_pint(int q, int N, int mc, int pin, const int32_t *cnodes, const double *DinvT,
                                 const double *H, const double *G, double *Zs, double *Ys, const double *r, double *z,
                                 int64_t ns, cudaStream_t s);
void launch_lu_inverse_batched(const double *LU, const int32_t *piv, int m, int batch, double *out, cudaStream_t s);

}  // namespace wrmg
