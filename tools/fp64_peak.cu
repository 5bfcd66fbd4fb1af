// FP64 FMA throughput of this B200 ("The FP64 peak must be
// measured first: a register-resident DFMA loop on all SMs, sustained >= 4 s").
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/fp64_peak tools/fp64_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(256) dfma_loop(double *out, int iters, double a, double b) {
  double x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-9 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 16; ++r)
#pragma unroll
      for (int i = 0; i < 8; ++i) x[i] = fma(x[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += x[i];
  if (s == 12345.678) out[0] = s;
}

// FP64 tensor-core MMA (mma.sync m8n8k4 f64): 8x8x4 = 256 FMA per warp instruction
__global__ void __launch_bounds__(256) dmma_loop(double *out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 0.999999;
  double c[4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i) c[i][0] = c[i][1] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 16; ++r)
#pragma unroll
      for (int i = 0; i < 4; ++i)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                     : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[0] = s;
}

int main() {
  int dev = 0, sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  double *out;
  cudaMalloc(&out, 8);
  const int blocks = sms * 8, threads = 256, iters = 4096;
  dfma_loop<<<blocks, threads>>>(out, 16, 0.999999, 1e-7);
  cudaDeviceSynchronize();
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  double best = 0, tot_ms = 0, tot_fl = 0;
  int reps = 0;
  while (tot_ms < 4000.0) {
    cudaEventRecord(a);
    dfma_loop<<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    double fl = 2.0 * blocks * threads * (double)iters * 16 * 8;
    best = fl / (ms * 1e-3) / 1e12 > best ? fl / (ms * 1e-3) / 1e12 : best;
    tot_ms += ms;
    tot_fl += fl;
    ++reps;
  }
  printf("{\"fp64_tflops_burst\": %.3f, \"fp64_tflops_sustained\": %.3f, \"seconds\": %.2f, \"sms\": %d, "
         "\"reps\": %d}\n",
         best, tot_fl / (tot_ms * 1e-3) / 1e12, tot_ms / 1e3, sms, reps);
  // DMMA
  dmma_loop<<<blocks, threads>>>(out, 16);
  cudaDeviceSynchronize();
  best = 0; tot_ms = 0; tot_fl = 0; reps = 0;
  while (tot_ms < 4000.0) {
    cudaEventRecord(a);
    dmma_loop<<<blocks, threads>>>(out, 1024);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    double fl = 2.0 * 256.0 * (blocks * threads / 32) * 1024.0 * 16 * 4;
    best = fl / (ms * 1e-3) / 1e12 > best ? fl / (ms * 1e-3) / 1e12 : best;
    tot_ms += ms;
    tot_fl += fl;
    ++reps;
  }
  printf("{\"dmma_tflops_burst\": %.3f, \"dmma_tflops_sustained\": %.3f, \"seconds\": %.2f}\n", best,
         tot_fl / (tot_ms * 1e-3) / 1e12, tot_ms / 1e3);
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
