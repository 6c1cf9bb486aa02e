// fp64 throughput probes on sm_100a: DFMA (CUDA cores) vs DMMA (mma.sync f64 shapes).
// Builder tool: measures the fp64 roofline denominator that MEASURED_PEAKS.json lacks.
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__global__ void dfma_kernel(double* out, int iters, double s) {
  double a[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = fma(a[i], s, 1e-7);
  }
  double r = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) r += a[i];
  if (r == 123.456) out[0] = r;
}

template <int K>
__device__ __forceinline__ void mma_f64(double (&d)[4], const double* a, const double* b);

template <>
__device__ __forceinline__ void mma_f64<4>(double (&d)[4], const double* a, const double* b) {
  asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
               : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3]) : "d"(a[0]), "d"(a[1]), "d"(b[0]));
}
template <>
__device__ __forceinline__ void mma_f64<8>(double (&d)[4], const double* a, const double* b) {
  asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
               : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3]) : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[0]), "d"(b[1]));
}
template <>
__device__ __forceinline__ void mma_f64<16>(double (&d)[4], const double* a, const double* b) {
  asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
               : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3])
               : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                 "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
}

template <int K>
__global__ void dmma_kernel(double* out, int iters) {
  double a[K / 2], b[K / 4];
#pragma unroll
  for (int i = 0; i < K / 2; ++i) a[i] = 1e-3 * (threadIdx.x + i);
#pragma unroll
  for (int i = 0; i < K / 4; ++i) b[i] = 1e-3 * (threadIdx.x - i);
  double d[8][4] = {};
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int t = 0; t < 8; ++t) mma_f64<K>(d[t], a, b);
  }
  double r = 0;
#pragma unroll
  for (int t = 0; t < 8; ++t) r += d[t][0] + d[t][1] + d[t][2] + d[t][3];
  if (r == 123.456) out[0] = r;
}

template <typename F>
float time_it(F f) {
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  f();
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(a);
    f();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  return best;
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out; CK(cudaMalloc(&out, 8));
  int iters = 1 << 16;
  for (int threads : {256, 512, 1024}) {
    for (int occ : {1, 2, 4}) {
      int blocks = sms * occ;
      float ms = time_it([&] { dfma_kernel<<<blocks, threads>>>(out, iters, 0.999999); });
      double flops = 2.0 * 8 * iters * (double)blocks * threads;
      printf("DFMA threads=%d blocks=%d: %.2f TFLOP/s\n", threads, blocks, flops / ms / 1e9);
    }
  }
  CK(cudaGetLastError());
  iters = 1 << 14;
  for (int threads : {128, 256, 512}) {
    for (int occ : {1, 2, 4}) {
      int blocks = sms * occ;
      float ms4 = time_it([&] { dmma_kernel<4><<<blocks, threads>>>(out, iters); });
      float ms8 = time_it([&] { dmma_kernel<8><<<blocks, threads>>>(out, iters); });
      float ms16 = time_it([&] { dmma_kernel<16><<<blocks, threads>>>(out, iters); });
      double warps = (double)blocks * threads / 32;
      double f4 = 2.0 * 16 * 8 * 4 * 8 * iters * warps;
      printf("DMMA threads=%d blocks=%d: m16n8k4 %.2f  m16n8k8 %.2f  m16n8k16 %.2f TFLOP/s\n", threads, blocks,
             f4 / ms4 / 1e9, 2 * f4 / ms8 / 1e9, 4 * f4 / ms16 / 1e9);
    }
  }
  CK(cudaGetLastError());
  return 0;
}
