// Micro-benchmark of the scatter options of the patch sweep (H8) on B200:
// FP64 atomics (RED.E.ADD.F64) in the sweep's access pattern (lane = slab, the
// two DG1 values 8 B apart: 32 lanes at a 16-byte stride) vs contiguous lanes,
// and a plain load-add-store read-modify-write.  81 M updates over a 303 MB
// vector (the C2 finest-level sweep), each element updated ~2.1 times.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o atomic_probe tools/atomic_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr long long kN = 303LL * 1000 * 1000 / 8;  // doubles
constexpr long long kOps = 81LL * 1000 * 1000;

__device__ __forceinline__ long long hashpos(long long w) {  // spread warps over the vector
  unsigned long long z = (unsigned long long)w * 0x9E3779B97F4A7C15ull;
  return (long long)(z % (unsigned long long)((kN - 64) / 64)) * 64;
}

// bulk reduction (TMA): each warp stages 64 doubles (512 B) in shared memory and one lane
// issues cp.reduce.async.bulk .add.f64 of the whole segment (UBLKRED), double-buffered
__global__ void kbulk(double *u, long long nwarp_ops) {
  __shared__ __align__(128) double buf[8][2][64];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const long long w0 = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
  int it = 0;
  for (long long wi = w0; wi < nwarp_ops; wi += nw, ++it) {
    const long long base = hashpos(wi);
    double *b = buf[w][it & 1];
    if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
    __syncwarp();
    b[2 * lane] = 1.0;
    b[2 * lane + 1] = 1.0;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncwarp();
    if (lane == 0) {
      asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f64 [%0], [%1], 512;" ::"l"(u + base),
                   "r"((unsigned)__cvta_generic_to_shared(b))
                   : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
  }
  if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

template <int MODE>
__global__ void k(double *u, long long nwarp_ops) {
  const int lane = threadIdx.x & 31;
  const long long w0 = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
  for (long long w = w0; w < nwarp_ops; w += nw) {
    const long long base = hashpos(w);
    if (MODE == 0) {  // sweep pattern: value a of slab lane at base + 2 lane + a
      atomicAdd(u + base + 2 * lane, 1.0);
      atomicAdd(u + base + 2 * lane + 1, 1.0);
    } else if (MODE == 1) {  // contiguous: 64 consecutive doubles in two instructions
      atomicAdd(u + base + lane, 1.0);
      atomicAdd(u + base + 32 + lane, 1.0);
    } else {  // plain read-modify-write, 16-byte lanes
      double2 *p = reinterpret_cast<double2 *>(u + base) + lane;
      double2 v = *p;
      v.x += 1.0;
      v.y += 1.0;
      *p = v;
    }
  }
}

int main() {
  double *u;
  cudaMalloc(&u, kN * sizeof(double));
  cudaMemset(u, 0, kN * sizeof(double));
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const long long nwarp_ops = kOps / 64;  // 64 element updates per warp iteration
  const char *names[4] = {"red_f64_stride16B(sweep pattern)", "red_f64_contiguous", "ld_add_st_rmw",
                          "bulk_reduce_512B(UBLKRED)"};
  for (int mode = 0; mode < 4; ++mode)
    for (int rep = 0; rep < 3; ++rep) {
      cudaEventRecord(a);
      if (mode == 0) k<0><<<148 * 8, 256>>>(u, nwarp_ops);
      if (mode == 1) k<1><<<148 * 8, 256>>>(u, nwarp_ops);
      if (mode == 2) k<2><<<148 * 8, 256>>>(u, nwarp_ops);
      if (mode == 3) kbulk<<<148 * 8, 256>>>(u, nwarp_ops);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (rep == 2) printf("%-36s %8.1f us  %7.1f G element-updates/s\n", names[mode], ms * 1e3, kOps / (ms * 1e-3) / 1e9);
    }
  printf("status %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
