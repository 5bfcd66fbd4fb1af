// Checks the register fragment layout of mma.sync.aligned.m8n8k4.row.col.f64
// assumed by kernels_kron.cu:
//   A (8x4):  a = A[lane >> 2][lane & 3]
//   B (4x8):  b = B[lane & 3][lane >> 2]
//   C (8x8):  c[e] = C[lane >> 2][2 (lane & 3) + e]
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k(const double *A, const double *B, double *C) {
  const int l = threadIdx.x;
  double a = A[(l >> 2) * 4 + (l & 3)];
  double b = B[(l & 3) * 8 + (l >> 2)];
  double c0 = 0, c1 = 0;
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
  C[(l >> 2) * 8 + 2 * (l & 3)] = c0;
  C[(l >> 2) * 8 + 2 * (l & 3) + 1] = c1;
}

int main() {
  double hA[32], hB[32], hC[64], ref[64];
  for (int i = 0; i < 32; ++i) {
    hA[i] = 1.0 + i;
    hB[i] = 0.5 * i - 3.0;
  }
  for (int i = 0; i < 8; ++i)
    for (int j = 0; j < 8; ++j) {
      double s = 0;
      for (int t = 0; t < 4; ++t) s += hA[i * 4 + t] * hB[t * 8 + j];
      ref[i * 8 + j] = s;
    }
  double *A, *B, *C;
  cudaMalloc(&A, 256);
  cudaMalloc(&B, 256);
  cudaMalloc(&C, 512);
  cudaMemcpy(A, hA, 256, cudaMemcpyHostToDevice);
  cudaMemcpy(B, hB, 256, cudaMemcpyHostToDevice);
  k<<<1, 32>>>(A, B, C);
  cudaMemcpy(hC, C, 512, cudaMemcpyDeviceToHost);
  double err = 0;
  for (int i = 0; i < 64; ++i) err = fmax(err, fabs(hC[i] - ref[i]));
  printf("{\"dmma_layout_max_abs_err\": %g, \"ok\": %s}\n", err, err == 0.0 ? "true" : "false");
  return err == 0.0 ? 0 : 1;
}
