// Dependent-chain latency probe (one warp): cycles per op for the FP64 / warp-collective
// instructions on the NS block-inversion panel's critical path.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double *out, long long *cyc, double x0, int n) {
  double x = x0 + threadIdx.x * 1e-9, y = 1.0 + threadIdx.x;
  unsigned u = threadIdx.x;
  long long t0, t1;
  // DFMA chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = fma(x, 0.999999, 1e-7);
  t1 = clock64(); cyc[0] = t1 - t0;
  // DMUL chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = x * 1.0000001;
  t1 = clock64(); cyc[1] = t1 - t0;
  // F2F f64->f32->u32 chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) { u = __float_as_uint((float)x) ^ u; x = (double)(u & 7) + x; }
  t1 = clock64(); cyc[2] = t1 - t0;
  // rcp.approx.f64 chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) { double r; asm volatile("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(y)); y = r + 1.5; }
  t1 = clock64(); cyc[3] = t1 - t0;
  // redux.sync.max chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) u = __reduce_max_sync(0xffffffffu, u + threadIdx.x);
  t1 = clock64(); cyc[4] = t1 - t0;
  // shfl (64-bit) chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) y = __shfl_sync(0xffffffffu, y, (threadIdx.x + 1) & 31) + 1.0;
  t1 = clock64(); cyc[5] = t1 - t0;
  // DADD chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) y = y + 1e-3;
  t1 = clock64(); cyc[6] = t1 - t0;
  // 1.0/x (compiler division) chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) y = 1.0 / y + 1.0;
  t1 = clock64(); cyc[7] = t1 - t0;
  // fmax shfl_xor butterfly step chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) y = fmax(y, __shfl_xor_sync(0xffffffffu, y, 1)) + 1e-9;
  t1 = clock64(); cyc[8] = t1 - t0;
  // hi-word integer key: LOP + max
  t0 = clock64();
  for (int i = 0; i < n; ++i) { u = max(u, (unsigned)(__double2hiint(x) & 0x7fffff80) | (u & 127)); x += (double)(u & 1); }
  t1 = clock64(); cyc[9] = t1 - t0;
  out[threadIdx.x] = x + y + u;
}
int main() {
  double *o; long long *c, h[16];
  cudaMalloc(&o, 32 * 8); cudaMalloc(&c, 16 * 8);
  const int n = 1000;
  for (int rep = 0; rep < 2; ++rep) k<<<1, 32>>>(o, c, 1.0, n);
  cudaMemcpy(h, c, 16 * 8, cudaMemcpyDeviceToHost);
  const char *nm[] = {"DFMA", "DMUL", "F2F f64->f32 + int", "rcp.approx.f64 + DADD", "REDUX.MAX + IADD", "SHFL64 + DADD",
                      "DADD", "1.0/x + DADD", "SHFL.BFLY64 + DMNMX + DADD", "hi-word key + IMNMX + DADD"};
  for (int i = 0; i < 10; ++i) printf("%-30s %6.1f cycles/iter\n", nm[i], (double)h[i] / n);
  return 0;
}
