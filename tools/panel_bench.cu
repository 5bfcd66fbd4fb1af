// Microbenchmark of the NS register-tiled Gauss-Jordan panel warp (k_ns_factor_rt's
// rt_panel): one warp factors 8-column panels of an M-row block held 3 rows per lane,
// variants of the pivot search / broadcast / reciprocal; prints cycles per column.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ double rcp_nr(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double e = fma(-x, r, 1.0);
  e = fma(e, e, e);
  r = fma(r, e, r);
  e = fma(-x, r, 1.0);
  r = fma(r, e, r);
  return x != 0.0 ? r : 0.0;
}

// V: 0 = as in kernels_ns.cu; 1 = high-word key; 2 = V1 + rcp after the broadcast;
//    3 = V1 + candidate row selected before the redux (one shuffle set, no uniform branch)
template <int M, int V>
__global__ void k(double *io, long long *cyc, int npanel, int m) {
  constexpr int RPL = (M + 31) / 32;
  const int lane = threadIdx.x;
  double P[RPL][8];
  for (int s = 0; s < RPL; ++s)
    for (int t = 0; t < 8; ++t) P[s][t] = io[(blockIdx.x * 97 + lane * 7 + s * 31 + t * 13) % 4096];
  unsigned elig = 0;
  for (int s = 0; s < RPL; ++s)
    if (lane + 32 * s < m) elig |= 1u << s;
  int mybi = 0;
  long long t0 = clock64();
  for (int pnl = 0; pnl < npanel; ++pnl) {
    if (pnl % 10 == 0) {
      elig = 0;
      for (int s = 0; s < RPL; ++s)
        if (lane + 32 * s < m) elig |= 1u << s;
    }
#pragma unroll
    for (int tc = 0; tc < 8; ++tc) {
      unsigned key = 0;
      double prow_v[8], pinv = 0.0;
      int bi, lp, sp;
      if (V == 3) {
        double cand[8];
#pragma unroll
        for (int t = 0; t < 8; ++t) cand[t] = P[0][t];
#pragma unroll
        for (int s = 0; s < RPL; ++s) {
          const double v = P[s][tc];
          const unsigned kk = ((elig >> s) & 1u)
                                  ? (((unsigned)__double2hiint(v) & 0x7FFFFF80u) | (unsigned)(127 - (lane + 32 * s)))
                                  : 0u;
          if (kk > key) {
            key = kk;
#pragma unroll
            for (int t = 0; t < 8; ++t) cand[t] = P[s][t];
          }
        }
        const double rl = rcp_nr(cand[tc]);
        const unsigned gk = __reduce_max_sync(0xffffffffu, key);
        bi = 127 - (int)(gk & 127u);
        lp = bi & 31;
        sp = bi >> 5;
#pragma unroll
        for (int t = 0; t < 8; ++t) prow_v[t] = __shfl_sync(0xffffffffu, cand[t], lp);
        pinv = __shfl_sync(0xffffffffu, rl, lp);
      } else if (V == 5) {
        __shared__ double bc[9];
        double rc[RPL];
#pragma unroll
        for (int s = 0; s < RPL; ++s) {
          const double v = P[s][tc];
          rc[s] = rcp_nr(v);
          const unsigned kk = ((elig >> s) & 1u)
                                  ? (((unsigned)__double2hiint(v) & 0x7FFFFF80u) | (unsigned)(255 - (lane + 32 * s)))
                                  : 0u;
          key = max(key, kk);
        }
        const unsigned gk = __reduce_max_sync(0xffffffffu, key);
        bi = 255 - (int)(gk & 255u);
        lp = bi & 31;
        sp = bi >> 5;
        if (lane == lp) {
#pragma unroll
          for (int s = 0; s < RPL; ++s)
            if (s == sp) {
#pragma unroll
              for (int t = 0; t < 8; ++t) bc[t] = P[s][t];
              bc[8] = rc[s];
            }
        }
        __syncwarp();
#pragma unroll
        for (int t = 0; t < 8; ++t) prow_v[t] = bc[t];
        pinv = bc[8];
        __syncwarp();
      } else {
        double rc[RPL];
#pragma unroll
        for (int s = 0; s < RPL; ++s) {
          const double v = P[s][tc];
          if (V != 2) rc[s] = rcp_nr(v);
          unsigned kk;
          if (V == 0)
            kk = ((elig >> s) & 1u) ? ((__float_as_uint((float)fabs(v)) & 0xFFFFFF00u) | (unsigned)(255 - (lane + 32 * s)))
                                    : 0u;
          else
            kk = ((elig >> s) & 1u) ? (((unsigned)__double2hiint(v) & 0x7FFFFF80u) | (unsigned)(255 - (lane + 32 * s)))
                                    : 0u;
          key = max(key, kk);
        }
        const unsigned gk = __reduce_max_sync(0xffffffffu, key);
        bi = 255 - (int)(gk & 255u);
        lp = bi & 31;
        sp = bi >> 5;
#pragma unroll
        for (int s = 0; s < RPL; ++s)
          if (s == sp) {
#pragma unroll
            for (int t = 0; t < 8; ++t) prow_v[t] = __shfl_sync(0xffffffffu, P[s][t], lp);
            if (V != 2) pinv = __shfl_sync(0xffffffffu, rc[s], lp);
          }
        if (V == 2) pinv = rcp_nr(prow_v[tc]);
      }
      if (V >= 4) {
        const bool isl = lane == lp;
        double keep[8];
        // the pivot row (slot sp of lane lp) before the update: prow_v scaled
#pragma unroll
        for (int s = 0; s < RPL; ++s) {
          const double frp = P[s][tc] * pinv;
#pragma unroll
          for (int t = 0; t < 8; ++t)
            if (t != tc) P[s][t] = fma(-frp, prow_v[t], P[s][t]);
          P[s][tc] = -frp;
        }
#pragma unroll
        for (int t = 0; t < 8; ++t) keep[t] = (t == tc) ? pinv : prow_v[t] * pinv;
        switch (sp) {
#pragma unroll
          case 0:
            for (int t = 0; t < 8; ++t) P[0][t] = isl ? keep[t] : P[0][t];
            break;
          case 1:
            for (int t = 0; t < 8; ++t) P[1 < RPL ? 1 : 0][t] = isl ? keep[t] : P[1 < RPL ? 1 : 0][t];
            break;
          default:
#pragma unroll
            for (int s = 2; s < RPL; ++s)
              if (s == sp)
#pragma unroll
                for (int t = 0; t < 8; ++t) P[s][t] = isl ? keep[t] : P[s][t];
            break;
        }
        if (isl) elig &= ~(1u << sp);
      } else {
      double newc[8];
#pragma unroll
      for (int t = 0; t < 8; ++t) newc[t] = (t == tc) ? pinv : prow_v[t] * pinv;
#pragma unroll
      for (int s = 0; s < RPL; ++s) {
        const double fr = P[s][tc];
#pragma unroll
        for (int t = 0; t < 8; ++t)
          if (t != tc) P[s][t] = fma(-fr, newc[t], P[s][t]);
        P[s][tc] = -fr * pinv;
      }
      if (lane == lp) {
#pragma unroll
        for (int s = 0; s < RPL; ++s)
          if (s == sp) {
#pragma unroll
            for (int t = 0; t < 8; ++t) P[s][t] = newc[t];
          }
        elig &= ~(1u << sp);
      }
      }
      if (lane == tc) mybi = bi;
    }
  }
  long long t1 = clock64();
  double acc = mybi;
  for (int s = 0; s < RPL; ++s)
    for (int t = 0; t < 8; ++t) acc += P[s][t];
  io[4096 + blockIdx.x * 32 + lane] = acc;
  if (lane == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int M, int V>
void run(double *io, long long *cyc, int nblk, int warpsper, const char *nm) {
  const int np = 40;
  k<M, V><<<nblk, 32>>>(io, cyc, np, M - 2);
  k<M, V><<<nblk, 32>>>(io, cyc, np, M - 2);
  cudaDeviceSynchronize();
  long long h[1024];
  cudaMemcpy(h, cyc, nblk * 8, cudaMemcpyDeviceToHost);
  double s = 0;
  for (int i = 0; i < nblk; ++i) s += h[i];
  printf("M=%3d %-34s %d warps/SM: %6.1f cycles/column\n", M, nm, warpsper, s / nblk / (np * 8));
}

int main() {
  double *io;
  long long *cyc;
  cudaMalloc(&io, (4096 + 1024 * 32) * 8);
  cudaMalloc(&cyc, 1024 * 8);
  double h[4096];
  for (int i = 0; i < 4096; ++i) h[i] = ((i * 2654435761u) % 1000) / 1000.0 - 0.5;
  cudaMemcpy(io, h, sizeof(h), cudaMemcpyHostToDevice);
  for (int per : {1}) {
    const int nb = 148 * per;
    run<80, 0>(io, cyc, nb, per, "V0 F2F key, spec. rcp per slot");
    run<80, 1>(io, cyc, nb, per, "V1 hi-word key, spec. rcp");
    run<80, 2>(io, cyc, nb, per, "V2 hi-word key, rcp after bcast");
    run<80, 3>(io, cyc, nb, per, "V3 cand. row before redux");
    run<80, 4>(io, cyc, nb, per, "V4 V1 + frp update, uniform fix");
    run<80, 5>(io, cyc, nb, per, "V5 V4 + smem broadcast");
    run<168, 0>(io, cyc, nb, per, "V0");
    run<168, 3>(io, cyc, nb, per, "V3");
    run<168, 4>(io, cyc, nb, per, "V4");
    run<168, 5>(io, cyc, nb, per, "V5");
  }
  return 0;
}
