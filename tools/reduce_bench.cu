// Latency of one "grid barrier + all-reduce of L values" step on sm_100a
// (builder tool for the panel / sample-QRCP per-column critical path).
//   A: every CTA reads all G partials of all L values (current panel scheme)
//   B: clusters of C CTAs: CTA r of a cluster reduces values v = r (mod C)
//      over all G partials and shares them through DSMEM (+ cluster barrier)
//   C: two barriers: CTA g reduces value g; every CTA then reads L values
//   D: barrier only
//   E: every CTA reads the same W doubles after the barrier (winner column)
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

__device__ __forceinline__ unsigned ld_rlx(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
struct Bar {
  unsigned* ctr;
  unsigned target = 0, nb;
  __device__ void sync() {
    __syncthreads();
    target += nb;
    if (threadIdx.x == 0) {
      asm volatile("fence.acq_rel.gpu;" ::: "memory");
      asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(ctr) : "memory");
      while ((int)(ld_rlx(ctr) - target) < 0) {
      }
      asm volatile("fence.acq_rel.gpu;" ::: "memory");
    }
    __syncthreads();
  }
};

constexpr int kT = 256;
constexpr int kMaxG = 152;

template <int MODE, int CL>
__global__ void __launch_bounds__(kT, 1) step_kernel(unsigned* ctr, double* part, double* red, int L, int iters,
                                                      double* sink) {
  __shared__ double vals[256];
  Bar b;
  b.ctr = ctr;
  b.nb = gridDim.x;
  const int G = gridDim.x, g = blockIdx.x, tid = threadIdx.x;
  double acc = 0.0;
  for (int it = 0; it < iters; ++it) {
    const int par = it & 1;
    // partials: value v of CTA g
    if (tid < L) part[((size_t)par * 256 + tid) * G + g] = acc + tid + g;
    if (MODE == 5) {
      cg::cluster_group cl = cg::this_cluster();
      // arrive: CTA-level sync, cluster-level sync, leader does the global atomic
      __syncthreads();
      cl.sync();
      b.target += gridDim.x / CL;
      if (cl.block_rank() == 0 && tid == 0) {
        asm volatile("fence.acq_rel.gpu;" ::: "memory");
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(ctr) : "memory");
        while ((int)(ld_rlx(ctr) - b.target) < 0) {
        }
        asm volatile("fence.acq_rel.gpu;" ::: "memory");
      }
      cl.sync();
    } else {
      b.sync();
    }
    if (MODE == 0) {
      for (int v0 = 0; v0 < L; v0 += kT / 4) {
        const int v = v0 + (tid >> 2), q = tid & 3;
        double x[kMaxG / 4];
        const double* src = part + ((size_t)par * 256 + v) * G;
#pragma unroll
        for (int i = 0; i < kMaxG / 4; ++i) {
          const int gi = q + 4 * i;
          x[i] = (v < L && gi < G) ? __ldcg(src + gi) : 0.0;
        }
        double s = 0.0;
#pragma unroll
        for (int i = 0; i < kMaxG / 4; ++i) s += x[i];
        s += __shfl_xor_sync(0xffffffffu, s, 2);
        s += __shfl_xor_sync(0xffffffffu, s, 1);
        if (v < L && q == 0) vals[v] = s;
      }
      __syncthreads();
    } else if (MODE == 1) {
      cg::cluster_group cl = cg::this_cluster();
      const int r = cl.block_rank();
      // my values: v = r + CL * j; 4 lanes per value
      const int nmine = (L - r + CL - 1) / CL;
      for (int j0 = 0; j0 < nmine; j0 += kT / 4) {
        const int j = j0 + (tid >> 2), q = tid & 3;
        const int v = r + CL * j;
        double x[kMaxG / 4];
        const double* src = part + ((size_t)par * 256 + v) * G;
#pragma unroll
        for (int i = 0; i < kMaxG / 4; ++i) {
          const int gi = q + 4 * i;
          x[i] = (j < nmine && gi < G) ? __ldcg(src + gi) : 0.0;
        }
        double s = 0.0;
#pragma unroll
        for (int i = 0; i < kMaxG / 4; ++i) s += x[i];
        s += __shfl_xor_sync(0xffffffffu, s, 2);
        s += __shfl_xor_sync(0xffffffffu, s, 1);
        if (j < nmine && q == 0) {
          for (int d = 0; d < CL; ++d) {
            double* dst = cl.map_shared_rank(vals, d);
            dst[v] = s;
          }
        }
      }
      cl.sync();
    } else if (MODE == 2) {
      if (g < L) {
        // CTA g reduces value g
        double s = 0.0;
        for (int i = tid; i < G; i += kT) s += __ldcg(part + ((size_t)par * 256 + g) * G + i);
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        __shared__ double ws[8];
        if ((tid & 31) == 0) ws[tid >> 5] = s;
        __syncthreads();
        if (tid == 0) {
          double t = 0;
          for (int w = 0; w < 8; ++w) t += ws[w];
          red[par * 256 + g] = t;
        }
      }
      b.sync();
      if (tid < L) vals[tid] = __ldcg(red + par * 256 + tid);
      __syncthreads();
    } else if (MODE == 5) {
      // (no reduction) barrier variant measured below
    } else if (MODE == 4) {
      if (tid < L) vals[tid] = __ldcg(part + (size_t)par * 256 * G + tid);
      __syncthreads();
    }
    acc += vals[tid % max(L, 1)] * 1e-30;
  }
  if (acc == -1.0) sink[0] = acc;
}

template <int MODE, int CL>
float run(int G, int L, int iters, unsigned* ctr, double* part, double* red, double* sink) {
  float best = 1e9;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int r = 0; r < 3; ++r) {
    cudaMemset(ctr, 0, 64);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(G);
    cfg.blockDim = dim3(kT);
    cudaLaunchAttribute at[2];
    int na = 0;
    at[na].id = cudaLaunchAttributeCooperative;
    at[na].val.cooperative = 1;
    ++na;
    if (CL > 1) {
      at[na].id = cudaLaunchAttributeClusterDimension;
      at[na].val.clusterDim.x = CL;
      at[na].val.clusterDim.y = 1;
      at[na].val.clusterDim.z = 1;
      ++na;
    }
    cfg.attrs = at;
    cfg.numAttrs = na;
    cudaGetLastError();
    cudaEventRecord(a);
    cudaError_t e = cudaLaunchKernelEx(&cfg, step_kernel<MODE, CL>, ctr, part, red, L, iters, sink);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    if (e != cudaSuccess || cudaGetLastError() != cudaSuccess) {
      printf("launch failed (%s) mode %d CL %d G %d\n", cudaGetErrorString(e), MODE, CL, G);
      return -1;
    }
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    best = ms < best ? ms : best;
  }
  return best * 1000.0f / iters;
}

int main() {
  unsigned* ctr;
  double *part, *red, *sink;
  cudaMalloc(&ctr, 64);
  cudaMalloc(&part, 2 * 256 * 152 * 8);
  cudaMalloc(&red, 2 * 256 * 8);
  cudaMalloc(&sink, 8);
  for (int cl : {2, 4, 8}) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(cl * 64);
    cfg.blockDim = dim3(kT);
    cudaLaunchAttribute at;
    at.id = cudaLaunchAttributeClusterDimension;
    at.val.clusterDim.x = cl;
    at.val.clusterDim.y = 1;
    at.val.clusterDim.z = 1;
    cfg.attrs = &at;
    cfg.numAttrs = 1;
    int ncl = 0;
    cudaError_t e = cl == 2   ? cudaOccupancyMaxActiveClusters(&ncl, step_kernel<1, 2>, &cfg)
                    : cl == 4 ? cudaOccupancyMaxActiveClusters(&ncl, step_kernel<1, 4>, &cfg)
                              : cudaOccupancyMaxActiveClusters(&ncl, step_kernel<1, 8>, &cfg);
    printf("cluster %d: max active clusters %d (%s)\n", cl, ncl, cudaGetErrorString(e));
  }
  const int iters = 2000;
  for (int G : {120, 132, 148}) {
    for (int L : {1, 32, 136}) {
      printf("G=%d L=%3d  A(all read) %.2f  C(2 barriers) %.2f  D(barrier) %.2f  E(same %d) %.2f us\n", G, L,
             run<0, 1>(G, L, iters, ctr, part, red, sink), run<2, 1>(G, L, iters, ctr, part, red, sink),
             run<3, 1>(G, L, iters, ctr, part, red, sink), L, run<4, 1>(G, L, iters, ctr, part, red, sink));
      printf("      H(barrier hier) cl2 %.2f", run<5, 2>(G, L, iters, ctr, part, red, sink));
      if (G <= 132) printf(" cl4 %.2f", run<5, 4>(G, L, iters, ctr, part, red, sink));
      if (G <= 120) printf(" cl8 %.2f", run<5, 8>(G, L, iters, ctr, part, red, sink));
      printf("\n");
      printf("      B cluster2 %.2f", run<1, 2>(G, L, iters, ctr, part, red, sink));
      if (G <= 132) printf("  cluster4 %.2f", run<1, 4>(G, L, iters, ctr, part, red, sink));
      if (G <= 120) printf("  cluster8 %.2f", run<1, 8>(G, L, iters, ctr, part, red, sink));
      printf(" us\n");
    }
  }
  return 0;
}
