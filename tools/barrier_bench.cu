// Grid-barrier latency probes on sm_100a (builder tool).
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

__device__ __forceinline__ unsigned ld_acq(const unsigned* p) { unsigned v; asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory"); return v; }
__device__ __forceinline__ unsigned ld_rlx(const unsigned* p) { unsigned v; asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory"); return v; }
__device__ __forceinline__ void st_rel(unsigned* p, unsigned v) { asm volatile("st.release.gpu.global.u32 [%0], %1;" :: "l"(p), "r"(v) : "memory"); }
__device__ __forceinline__ unsigned atom_add_rel(unsigned* p, unsigned v) { unsigned o; asm volatile("atom.add.release.gpu.global.u32 %0, [%1], %2;" : "=r"(o) : "l"(p), "r"(v) : "memory"); return o; }
__device__ __forceinline__ unsigned atom_add_acqrel(unsigned* p, unsigned v) { unsigned o; asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], %2;" : "=r"(o) : "l"(p), "r"(v) : "memory"); return o; }
__device__ __forceinline__ void fence_acqrel() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }

// V1: current libsqr barrier
__global__ void v1(unsigned* bar, int iters, double* sink) {
  __shared__ unsigned s0; if (threadIdx.x == 0) s0 = ld_acq(bar + 1); __syncthreads();
  unsigned sense = s0, nb = gridDim.x;
  double acc = 0;
  for (int i = 0; i < iters; ++i) {
    __syncthreads(); sense ^= 1u;
    if (threadIdx.x == 0) {
      __threadfence();
      unsigned old = atomicAdd(bar, 1u);
      if (old == nb - 1) { atomicExch(bar, 0u); __threadfence(); st_rel(bar + 1, sense); }
      else while (ld_acq(bar + 1) != sense) {}
      __threadfence();
    }
    __syncthreads();
    acc += i;
  }
  if (acc == -1) sink[0] = acc;
}
// V2: monotonic counter, release-add arrive, relaxed poll, one acquire fence
__global__ void v2(unsigned* bar, int iters, double* sink) {
  unsigned target = 0; const unsigned nb = gridDim.x; double acc = 0;  // counter zeroed before every launch
  // all CTAs must agree on base: guaranteed since counter is a multiple of nb between launches
  for (int i = 0; i < iters; ++i) {
    __syncthreads();
    target += nb;
    if (threadIdx.x == 0) {
      atom_add_rel(bar, 1u);
      while ((int)(ld_rlx(bar) - target) < 0) {}
      fence_acqrel();
    }
    __syncthreads();
    acc += i;
  }
  if (acc == -1) sink[0] = acc;
}
// V3: cooperative groups
__global__ void v3(int iters, double* sink) {
  cg::grid_group g = cg::this_grid(); double acc = 0;
  for (int i = 0; i < iters; ++i) { g.sync(); acc += i; }
  if (acc == -1) sink[0] = acc;
}
// V4: flag-per-CTA gather by CTA 0, broadcast by one word
__global__ void v4(unsigned* flags, int iters, double* sink) {
  const unsigned nb = gridDim.x; double acc = 0;
  __shared__ unsigned base; if (threadIdx.x == 0) base = ld_acq(flags + 1024); __syncthreads();
  unsigned gen = base;
  for (int i = 0; i < iters; ++i) {
    __syncthreads(); ++gen;
    if (blockIdx.x == 0) {
      if (threadIdx.x < nb && threadIdx.x > 0) { while ((int)(ld_rlx(flags + threadIdx.x * 32) - gen) < 0) {} }
      __syncthreads();
      if (threadIdx.x == 0) { fence_acqrel(); st_rel(flags + 1024, gen); }
    } else if (threadIdx.x == 0) {
      st_rel(flags + blockIdx.x * 32, gen);
      while ((int)(ld_rlx(flags + 1024) - gen) < 0) {}
      fence_acqrel();
    }
    __syncthreads();
    acc += i;
  }
  if (acc == -1) sink[0] = acc;
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned* bar; cudaMalloc(&bar, 1 << 20); cudaMemset(bar, 0, 1 << 20);
  double* sink; cudaMalloc(&sink, 8);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  int iters = 2000;
  for (int G : {16, 74, 148}) {
    for (int v = 1; v <= 4; ++v) {
      float best = 1e9;
      for (int r = 0; r < 3; ++r) {
        cudaMemset(bar, 0, 1 << 20);
        cudaEventRecord(a);
        if (v == 1) { void* args[] = {&bar, &iters, &sink}; cudaLaunchCooperativeKernel((void*)v1, G, 256, args, 0, 0); }
        if (v == 2) { void* args[] = {&bar, &iters, &sink}; cudaLaunchCooperativeKernel((void*)v2, G, 256, args, 0, 0); }
        if (v == 3) { void* args[] = {&iters, &sink}; cudaLaunchCooperativeKernel((void*)v3, G, 256, args, 0, 0); }
        if (v == 4) { void* args[] = {&bar, &iters, &sink}; cudaLaunchCooperativeKernel((void*)v4, G, 256, args, 0, 0); }
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b); if (ms < best) best = ms;
      }
      cudaError_t e = cudaGetLastError();
      printf("G=%3d v%d: %.3f us/barrier %s\n", G, v, best * 1000.0 / iters, e ? cudaGetErrorString(e) : ""); fflush(stdout);
    }
  }
  return 0;
}
