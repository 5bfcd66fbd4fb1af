// Space-time residual (H6) with stencil classes.
//
//   r_n = b_n - [(C+E0) (x) M + Mt (x) kappa K] u_n + (E1 (x) M) u_{n-1}     (eq. heatfem, R1-R3)
//   constrained rows: r = b - u                                               (R5)
//
// Rows of the structured lattice whose surrounding cells are identical have
// identical CSR rows (same neighbour offsets, same values): wrmg_setup groups
// them into stencil classes (host_plan.cu) whose (offset, M, kappa K) tables
// travel as a kernel parameter (constant bank, broadcast), so the hot loop reads
// no indices and no matrix values from memory.  A CTA owns an 8x8 tile of rows
// and walks the slabs in 32-slab chunks; each chunk of u (tile + k-wide halo)
// is staged once in shared memory with cp.async.  Warp = one row x 32 slabs,
// lane = slab: the jump term (M u)_{n-1}[q] is lane n-1's own accumulator,
// passed with a shuffle; lane 0 takes lane 31's value of the previous chunk.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <map>
#include <mutex>
#include <tuple>

#include "internal.h"

namespace wrmg {
namespace {

constexpr int TR = 8;  // tile rows per direction

struct TMr {
  double CE[16], Mt[16];
};

__device__ __forceinline__ void cp_async16(void *smem, const void *gmem) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::); }

template <int NQ>
__global__ void __launch_bounds__(256) k_residual_cls(int k, int Lx, int Ly, int N,
                                                      const uint8_t *__restrict__ rcls,
                                                      const double *__restrict__ u, const double *__restrict__ b,
                                                      double *__restrict__ r, TMr tm, const StencilTab T, int apply) {
  extern __shared__ __align__(16) double su[];
  __shared__ double prevq[TR * TR];
  constexpr int W = 32 * NQ;  // doubles per staged node (one chunk)
  const int64_t NT = (int64_t)N * NQ;
  const int ntx = (Lx + TR - 1) / TR;
  const int tx0 = (blockIdx.x % ntx) * TR, ty0 = (blockIdx.x / ntx) * TR;
  const int RW = TR + 2 * k;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  if (tid < TR * TR) prevq[tid] = 0.0;
  const int nchunk = (N + 31) / 32;
  for (int ch = 0; ch < nchunk; ++ch) {
    const int n0 = ch * 32;
    const int nv = min(32, N - n0) * NQ;  // valid doubles per node in this chunk
    __syncthreads();                      // previous chunk fully consumed
    // stage u: one warp per node, 16-byte pieces (2 doubles), NQ*32 doubles per node
    constexpr int PIECES = W / 2;
    for (int node = wid; node < RW * RW; node += 8) {
      const int I = tx0 - k + node % RW, J = ty0 - k + node / RW;
      const bool in = I >= 0 && I < Lx && J >= 0 && J < Ly;
      const double *srcn = u + ((int64_t)J * Lx + I) * NT + (int64_t)n0 * NQ;
      const bool al = in && ((reinterpret_cast<uintptr_t>(srcn) & 15) == 0);
      for (int pc = lane; pc < PIECES; pc += 32) {
        double *dst = su + node * W + 2 * pc;
        if (al && 2 * pc + 1 < nv) {
          cp_async16(dst, srcn + 2 * pc);
        } else if (in && 2 * pc < nv) {
          dst[0] = srcn[2 * pc];
          dst[1] = (2 * pc + 1 < nv) ? srcn[2 * pc + 1] : 0.0;
        } else {
          dst[0] = 0.0;
          dst[1] = 0.0;
        }
      }
    }
    cp_async_wait_all();
    __syncthreads();
    const int n = n0 + lane;
    const bool valid = n < N;
    for (int rr = wid; rr < TR * TR; rr += 8) {
      const int I = tx0 + rr % TR, J = ty0 + rr / TR;
      if (I >= Lx || J >= Ly) continue;
      const int64_t i = (int64_t)J * Lx + I;
      const int64_t base = i * NT + (int64_t)n * NQ;
      const double *own = su + ((J - ty0 + k) * RW + (I - tx0 + k)) * W + lane * NQ;
      const int cls = rcls[i];
      // issue the b loads first: their DRAM latency overlaps the stencil loop
      double bv[NQ];
#pragma unroll
      for (int a = 0; a < NQ; ++a) bv[a] = (valid && !apply) ? __ldg(b + base + a) : 0.0;
      if (cls >= T.ncls) {  // constrained row (identity)
        if (valid)
#pragma unroll
          for (int a = 0; a < NQ; ++a) r[base + a] = apply ? own[a] : bv[a] - own[a];
        continue;
      }
      double am[NQ], ak[NQ];
#pragma unroll
      for (int a = 0; a < NQ; ++a) am[a] = ak[a] = 0.0;
      const int cnt = T.cnt[cls];
#pragma unroll 8
      for (int e = 0; e < cnt; ++e) {
        const double *ul = own + T.off[cls][e];
        const double mv = T.m[cls][e], kv = T.kk[cls][e];
        if constexpr (NQ == 2) {
          const double2 uv = *reinterpret_cast<const double2 *>(ul);
          am[0] = fma(mv, uv.x, am[0]);
          am[1] = fma(mv, uv.y, am[1]);
          ak[0] = fma(kv, uv.x, ak[0]);
          ak[1] = fma(kv, uv.y, ak[1]);
        } else {
#pragma unroll
          for (int a = 0; a < NQ; ++a) {
            const double x = ul[a];
            am[a] = fma(mv, x, am[a]);
            ak[a] = fma(kv, x, ak[a]);
          }
        }
      }
      // jump: (M u)_{n-1}[q] is lane n-1's am[q]; lane 0 uses the previous chunk
      double jm = __shfl_up_sync(0xffffffffu, am[NQ - 1], 1);
      if (lane == 0) jm = prevq[rr];
      const double last = __shfl_sync(0xffffffffu, am[NQ - 1], 31);
      if (valid) {
#pragma unroll
        for (int a = 0; a < NQ; ++a) {
          double acc = bv[a];
#pragma unroll
          for (int c = 0; c < NQ; ++c) acc -= tm.CE[a * NQ + c] * am[c] + tm.Mt[a * NQ + c] * ak[c];
          if (a == 0 && n > 0) acc += jm;
          r[base + a] = apply ? -acc : acc;  // apply: y = A u = -(0 - A u)
        }
      }
      __syncwarp();
      if (lane == 0) prevq[rr] = last;
    }
  }
}


// ---- TMA variant: the (tile + halo) x 32-slab box of u is one 3D tensor-map copy
// (dims: time values, I, J), out-of-lattice halo and slabs beyond N zero-filled by
// the TMA unit; completion through an mbarrier transaction count.
__device__ __forceinline__ void mbar_init(uint64_t *bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"((unsigned)__cvta_generic_to_shared(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(
                   (unsigned)__cvta_generic_to_shared(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, unsigned parity) {
  const unsigned a = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(a),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_3d(void *dst, const CUtensorMap *map, int c0, int c1, int c2, uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
      "[%5];\n" ::"r"((unsigned)__cvta_generic_to_shared(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"((unsigned)__cvta_generic_to_shared(bar))
      : "memory");
}

template <int NQ>
__global__ void __launch_bounds__(256, 2) k_residual_tma(const __grid_constant__ CUtensorMap umap, int k, int Lx,
                                                         int Ly, int N, const uint8_t *__restrict__ rcls,
                                                         const double *__restrict__ b, double *__restrict__ r, TMr tm,
                                                         const StencilTab T, int apply) {
  extern __shared__ __align__(128) double su[];
  __shared__ __align__(8) uint64_t bar;
  __shared__ double prevq[TR * TR];
  // class tables behind the u tile in dynamic shared memory (broadcast loads, no LDC)
  constexpr int W = 32 * NQ;
  const int64_t NT = (int64_t)N * NQ;
  const int ntx = (Lx + TR - 1) / TR;
  const int tx0 = (blockIdx.x % ntx) * TR, ty0 = (blockIdx.x / ntx) * TR;
  const int RW = TR + 2 * k;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const unsigned bytes = (unsigned)(RW * RW * W * sizeof(double));
  double2 *smk = reinterpret_cast<double2 *>(su + RW * RW * W);
  int *soff = reinterpret_cast<int *>(smk + T.ncls * kStencilMaxE);
  for (int e = tid; e < T.ncls * kStencilMaxE; e += blockDim.x) {
    const int c = e / kStencilMaxE, x = e - c * kStencilMaxE;
    smk[e] = make_double2(T.m[c][x], T.kk[c][x]);
    soff[e] = T.off[c][x];
  }
  if (tid < TR * TR) prevq[tid] = 0.0;
  if (tid == 0) {
    mbar_init(&bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  const int nchunk = (N + 31) / 32;
  for (int ch = 0; ch < nchunk; ++ch) {
    const int n0 = ch * 32;
    if (ch) __syncthreads();  // the previous chunk is fully consumed
    if (tid == 0) {
      asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
      mbar_expect_tx(&bar, bytes);
      tma_load_3d(su, &umap, n0 * NQ, tx0 - k, ty0 - k, &bar);
    }
    mbar_wait(&bar, ch & 1);
    const int n = n0 + lane;
    const bool valid = n < N;
    for (int rr = wid; rr < TR * TR; rr += 8) {
      const int I = tx0 + rr % TR, J = ty0 + rr / TR;
      if (I >= Lx || J >= Ly) continue;
      const int64_t i = (int64_t)J * Lx + I;
      const int64_t base = i * NT + (int64_t)n * NQ;
      const double *own = su + ((J - ty0 + k) * RW + (I - tx0 + k)) * W + lane * NQ;
      const int cls = __shfl_sync(0xffffffffu, (int)rcls[i], 0);
      double bv[NQ];
#pragma unroll
      for (int a = 0; a < NQ; ++a) bv[a] = (valid && !apply) ? __ldg(b + base + a) : 0.0;
      if (cls >= T.ncls) {  // constrained row (identity)
        if (valid)
#pragma unroll
          for (int a = 0; a < NQ; ++a) r[base + a] = apply ? own[a] : bv[a] - own[a];
        continue;
      }
      double am[NQ], ak[NQ];
#pragma unroll
      for (int a = 0; a < NQ; ++a) am[a] = ak[a] = 0.0;
      const int cnt = T.cnt[cls];  // padded to a multiple of 4 with zero entries
      const double2 *mk = smk + cls * kStencilMaxE;
      const int *of = soff + cls * kStencilMaxE;
      for (int e0 = 0; e0 < cnt; e0 += 4) {
#pragma unroll
        for (int e = e0; e < e0 + 4; ++e) {
          const double *ul = own + of[e];
          const double2 w2 = mk[e];
          const double mv = w2.x, kv = w2.y;
          if constexpr (NQ == 2) {
            const double2 uv = *reinterpret_cast<const double2 *>(ul);
            am[0] = fma(mv, uv.x, am[0]);
            am[1] = fma(mv, uv.y, am[1]);
            ak[0] = fma(kv, uv.x, ak[0]);
            ak[1] = fma(kv, uv.y, ak[1]);
          } else {
#pragma unroll
            for (int a = 0; a < NQ; ++a) {
              const double x = ul[a];
              am[a] = fma(mv, x, am[a]);
              ak[a] = fma(kv, x, ak[a]);
            }
          }
        }
      }
      double jm = __shfl_up_sync(0xffffffffu, am[NQ - 1], 1);
      if (lane == 0) jm = prevq[rr];
      const double last = __shfl_sync(0xffffffffu, am[NQ - 1], 31);
      if (valid) {
#pragma unroll
        for (int a = 0; a < NQ; ++a) {
          double acc = bv[a];
#pragma unroll
          for (int c = 0; c < NQ; ++c) acc -= tm.CE[a * NQ + c] * am[c] + tm.Mt[a * NQ + c] * ak[c];
          if (a == 0 && n > 0) acc += jm;
          r[base + a] = apply ? -acc : acc;
        }
      }
      __syncwarp();
      if (lane == 0) prevq[rr] = last;
    }
  }
}


// ---- L1 variant: no staging.  Warp = one row x 32 slabs (lane = slab); the
// neighbour time histories are read straight from global memory (LDG.128,
// L1-allocating).  A CTA walks an 8x8 tile of rows so the tile's neighbourhood
// stays L1-resident; with no shared memory and ~40 registers an SM holds 64
// warps, each with up to `cnt` independent loads in flight.
template <int NQ, int TRL>
__global__ void __launch_bounds__(256) k_residual_l1(int Lx, int Ly, int N, const uint8_t *__restrict__ rcls,
                                                     const double *__restrict__ u, const double *__restrict__ b,
                                                     double *__restrict__ r, TMr tm, const StencilTab T, int apply,
                                                     const int64_t *__restrict__ goff) {
  const int64_t NT = (int64_t)N * NQ;
  const int ntx = (Lx + TRL - 1) / TRL;
  const int tx0 = (blockIdx.x % ntx) * TRL, ty0 = (blockIdx.x / ntx) * TRL;
  const int n0 = blockIdx.y * 32;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int n = n0 + lane;
  const bool valid = n < N;
  const int ns = valid ? n : N - 1;  // clamp loads of idle lanes
  for (int rr = wid; rr < TRL * TRL; rr += 8) {
    const int I = tx0 + rr % TRL, J = ty0 + rr / TRL;
    if (I >= Lx || J >= Ly) continue;
    const int64_t i = (int64_t)J * Lx + I;
    const int64_t base = i * NT + (int64_t)ns * NQ;
    const int cls = __ldg(rcls + i);
    double bv[NQ];
#pragma unroll
    for (int a = 0; a < NQ; ++a) bv[a] = apply ? 0.0 : __ldg(b + base + a);
    if (cls >= T.ncls) {
      if (valid)
#pragma unroll
        for (int a = 0; a < NQ; ++a) r[base + a] = apply ? __ldg(u + base + a) : bv[a] - __ldg(u + base + a);
      continue;
    }
    double am[NQ], ak[NQ], ap = 0.0;
#pragma unroll
    for (int a = 0; a < NQ; ++a) am[a] = ak[a] = 0.0;
    const double *ub = u + base;
    const int cnt = T.cnt[cls];
    const int64_t *go = goff + cls * kStencilMaxE;
    for (int e0 = 0; e0 < cnt; e0 += 4) {
#pragma unroll
      for (int e = e0; e < e0 + 4; ++e) {
        const double *ul = ub + __ldg(go + e);
        const double mv = T.m[cls][e], kv = T.kk[cls][e];
        if constexpr (NQ == 2) {
          const double2 uv = __ldg(reinterpret_cast<const double2 *>(ul));
          am[0] = fma(mv, uv.x, am[0]);
          am[1] = fma(mv, uv.y, am[1]);
          ak[0] = fma(kv, uv.x, ak[0]);
          ak[1] = fma(kv, uv.y, ak[1]);
        } else {
#pragma unroll
          for (int a = 0; a < NQ; ++a) {
            const double x = __ldg(ul + a);
            am[a] = fma(mv, x, am[a]);
            ak[a] = fma(kv, x, ak[a]);
          }
        }
        if (lane == 0 && n > 0) ap = fma(mv, __ldg(ul - 1), ap);  // (M u)_{n0-1}[q] for the chunk's first slab
      }
    }
    double jm = __shfl_up_sync(0xffffffffu, am[NQ - 1], 1);
    if (lane == 0) jm = ap;
    if (valid) {
#pragma unroll
      for (int a = 0; a < NQ; ++a) {
        double acc = bv[a];
#pragma unroll
        for (int c = 0; c < NQ; ++c) acc -= tm.CE[a * NQ + c] * am[c] + tm.Mt[a * NQ + c] * ak[c];
        if (a == 0 && n > 0) acc += jm;
        r[base + a] = apply ? -acc : acc;
      }
    }
  }
}


PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (PFN_cuTensorMapEncodeTiled_v12000)p;
  });
  return fn;
}

}  // namespace

// Tensor map of a waveform-major vector: dims (NT, Lx, Ly), box (boxT, RW, RWy).
// Encoded maps are cached per (pointer, shape, box) under a lock: strips run
// several contexts as host threads of one process (loopback transport).
bool umap_for(const double *u, int64_t NT, int Lx, int Ly, int boxT, int RW, CUtensorMap *out, int RWy) {
  if (RWy < 0) RWy = RW;
  static std::mutex mu;
  static std::map<std::tuple<const double *, int64_t, int, int, int, int, int>, CUtensorMap> cache;
  auto key = std::make_tuple(u, NT, Lx, Ly, boxT, RW, RWy);
  std::lock_guard<std::mutex> lk(mu);
  auto it = cache.find(key);
  if (it != cache.end()) {
    *out = it->second;
    return true;
  }
  auto enc = get_encode();
  if (!enc || (NT * 8) % 16 || (reinterpret_cast<uintptr_t>(u) & 15)) return false;
  cuuint64_t dims[3] = {(cuuint64_t)NT, (cuuint64_t)Lx, (cuuint64_t)Ly};
  cuuint64_t strides[2] = {(cuuint64_t)NT * 8, (cuuint64_t)NT * 8 * Lx};
  cuuint32_t box[3] = {(cuuint32_t)boxT, (cuuint32_t)RW, (cuuint32_t)RWy};
  cuuint32_t es[3] = {1, 1, 1};
  CUtensorMap m;
  CUresult rc = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double *>(u), dims, strides, box, es,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (rc != CUDA_SUCCESS) return false;
  if (cache.size() > 4096) cache.clear();
  cache.emplace(key, m);
  *out = m;
  return true;
}

namespace {

// Fill the class tables from the assembled CSR of each class's representative row.
__global__ void k_gather_classes(int ncls, const int32_t *__restrict__ rep, int Lx, const int32_t *__restrict__ rowptr,
                                 const int32_t *__restrict__ col, const double *__restrict__ Mv,
                                 const double *__restrict__ Kv, int maxe, int32_t *__restrict__ cnt,
                                 int32_t *__restrict__ dI, int32_t *__restrict__ dJ, double *__restrict__ m,
                                 double *__restrict__ kk) {
  const int c = blockIdx.x;
  if (c >= ncls) return;
  const int64_t i = rep[c];
  const int e0 = rowptr[i], ne = rowptr[i + 1] - e0;
  if (threadIdx.x == 0) cnt[c] = ne;
  const int I = (int)(i % Lx), J = (int)(i / Lx);
  for (int e = threadIdx.x; e < ne && e < maxe; e += blockDim.x) {
    const int j = col[e0 + e];
    dI[c * maxe + e] = j % Lx - I;
    dJ[c * maxe + e] = j / Lx - J;
    m[c * maxe + e] = Mv[e0 + e];
    kk[c * maxe + e] = Kv[e0 + e];
  }
}

}  // namespace

void launch_gather_classes(const Level &L, int32_t *scratch_i, double *scratch_d, cudaStream_t s) {
  const int nc = (int)L.h_cls_rep.size();
  k_gather_classes<<<nc, 64, 0, s>>>(nc, scratch_i, L.Lx, L.A.rowptr, L.A.col, L.A.val, L.A.val2, kStencilMaxE,
                                     scratch_i + nc, scratch_i + 2 * nc, scratch_i + 2 * nc + nc * kStencilMaxE,
                                     scratch_d, scratch_d + nc * kStencilMaxE);
  ++g_launches;
}

bool launch_residual_cls(const Level &L, int q, int N, const Temporal &tm, const double *u, const double *b,
                         double *r, cudaStream_t s) {
  const int apply = b == nullptr;
  if (!L.stencil_ok) return false;
  if (L.goff && L.nnode < 50000) {  // small levels: no staging latency; large levels: TMA tiles below
    TMr t{};
    for (int e = 0; e < tm.nq * tm.nq; ++e) {
      t.CE[e] = tm.CE[e];
      t.Mt[e] = tm.Mt[e];
    }
    // 8x8-row tiles, or 4x4 when that leaves fewer than 4 CTAs per SM (the
    // coarsest levels are latency-bound: more, shorter CTAs)
    const int nchunk = (N + 31) / 32;
    const bool small = (int64_t)((L.Lx + TR - 1) / TR) * ((L.Ly + TR - 1) / TR) * nchunk < 4 * num_sms();
    const int tr = small ? 4 : TR;
    const int ntx = (L.Lx + tr - 1) / tr, nty = (L.Ly + tr - 1) / tr;
    dim3 grid(ntx * nty, nchunk);
#define WRMG_RL(NQ)                                                                                             \
  if (small)                                                                                                   \
    k_residual_l1<NQ, 4><<<grid, 256, 0, s>>>(L.Lx, L.Ly, N, L.rcls, u, b, r, t, L.stencil, apply, L.goff);      \
  else                                                                                                         \
    k_residual_l1<NQ, TR><<<grid, 256, 0, s>>>(L.Lx, L.Ly, N, L.rcls, u, b, r, t, L.stencil, apply, L.goff);
    switch (q) {
      case 0: WRMG_RL(1) break;
      case 1: WRMG_RL(2) break;
      case 2: WRMG_RL(3) break;
      default: WRMG_RL(4) break;
    }
#undef WRMG_RL
    ++g_launches;
    return true;
  }
  const int k = (L.Lx - 1) / L.nx;
  const int ntx = (L.Lx + TR - 1) / TR, nty = (L.Ly + TR - 1) / TR;
  const int RW = TR + 2 * k;
  TMr t{};
  for (int e = 0; e < tm.nq * tm.nq; ++e) {
    t.CE[e] = tm.CE[e];
    t.Mt[e] = tm.Mt[e];
  }
  const size_t smem = (size_t)RW * RW * 32 * (q + 1) * sizeof(double);
  if (smem > 200 * 1024) return false;
  const size_t tab = (size_t)L.stencil.ncls * kStencilMaxE * (sizeof(double2) + sizeof(int));
  const bool tma_fits = smem + tab <= 220 * 1024;  // u tile + class tables in dynamic shared memory
  CUtensorMap umap;
  if (tma_fits && RW <= 256 && 32 * (q + 1) <= 256 && umap_for(u, (int64_t)N * (q + 1), L.Lx, L.Ly, 32 * (q + 1), RW, &umap)) {
#define WRMG_RT(NQ)                                                                                          \
    {                                                                                                        \
      smem_optin((const void *)k_residual_tma<NQ>, (int)(smem + tab));                                                                                                      \
      k_residual_tma<NQ><<<ntx * nty, 256, smem + tab, s>>>(umap, k, L.Lx, L.Ly, N, L.rcls, b, r, t,          \
                                                            L.stencil,                                       \
                                                      apply);                                                \
      ++g_launches;                                                                                          \
      return true;                                                                                           \
    }
    switch (q) {
      case 0: WRMG_RT(1);
      case 1: WRMG_RT(2);
      case 2: WRMG_RT(3);
      default: WRMG_RT(4);
    }
#undef WRMG_RT
  }
#define WRMG_RC(NQ)                                                                                          \
  {                                                                                                          \
    smem_optin((const void *)k_residual_cls<NQ>, 200 * 1024);                                                                                                        \
    k_residual_cls<NQ><<<ntx * nty, 256, smem, s>>>(k, L.Lx, L.Ly, N, L.rcls, u, b, r, t, L.stencil, apply);        \
    ++g_launches;                                                                                            \
    return true;                                                                                             \
  }
  switch (q) {
    case 0: WRMG_RC(1);
    case 1: WRMG_RC(2);
    case 2: WRMG_RC(3);
    default: WRMG_RC(4);
  }
#undef WRMG_RC
}

}  // namespace wrmg
