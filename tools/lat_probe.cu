// Latency microbenchmarks on the GPU (builder tool): dependent-chain cycles of
// DFMA / DADD / shfl(double) / LDS / bar.sync(224 threads) / fp64 sqrt + div,
// one warp (or one CTA for bar.sync), clock64 around N iterations.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/lat_probe tools/lat_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k(double* out, long long* cyc, double a, double b, int n) {
  __shared__ double sm[1024];
  const int tid = threadIdx.x;
  for (int i = tid; i < 1024; i += blockDim.x) sm[i] = (i * 7 + 3) % 1024;
  __syncthreads();
  double x = a + tid;
  long long t0, t1;
  // DFMA chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = fma(x, a, b);
  t1 = clock64();
  if (tid == 0) cyc[0] = t1 - t0;
  // DADD chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = x + b;
  t1 = clock64();
  if (tid == 0) cyc[1] = t1 - t0;
  // shfl(double) chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = __shfl_xor_sync(0xffffffffu, x, 1) + b;
  t1 = clock64();
  if (tid == 0) cyc[2] = t1 - t0;
  // LDS chain (pointer chase through smem values)
  int p = tid & 1023;
  t0 = clock64();
  for (int i = 0; i < n; ++i) p = (int)sm[p];
  t1 = clock64();
  if (tid == 0) cyc[3] = t1 - t0;
  x += p;
  // bar.sync 1, 224 (warps 0..6)
  if (tid < 224) {
    t0 = clock64();
    for (int i = 0; i < n; ++i) asm volatile("bar.sync 1, 224;\n" ::: "memory");
    t1 = clock64();
    if (tid == 0) cyc[4] = t1 - t0;
  }
  __syncthreads();
  // sqrt chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = sqrt(x + 2.0);
  t1 = clock64();
  if (tid == 0) cyc[5] = t1 - t0;
  // div chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = 3.0 / (x + 1.5);
  t1 = clock64();
  if (tid == 0) cyc[6] = t1 - t0;
  // drcp_rn chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = __drcp_rn(x + 1.5);
  t1 = clock64();
  if (tid == 0) cyc[7] = t1 - t0;
  // __syncthreads (256)
  t0 = clock64();
  for (int i = 0; i < n; ++i) __syncthreads();
  t1 = clock64();
  if (tid == 0) cyc[8] = t1 - t0;
  // volatile smem flag ping-pong between warp 0 and warp 1 (one round trip)
  volatile int* flag = reinterpret_cast<volatile int*>(sm);
  if (tid == 0) flag[0] = 0;
  __syncthreads();
  t0 = clock64();
  if (tid == 0) {
    for (int i = 0; i < n; ++i) {
      flag[0] = 2 * i + 1;
      while (flag[0] != 2 * i + 2) {
      }
    }
  } else if (tid == 32) {
    for (int i = 0; i < n; ++i) {
      while (flag[0] != 2 * i + 1) {
      }
      flag[0] = 2 * i + 2;
    }
  }
  t1 = clock64();
  if (tid == 0) cyc[9] = t1 - t0;
  out[tid] = x;
}

int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 256 * 8);
  cudaMallocManaged(&cyc, 16 * 8);
  const int n = 1000;
  k<<<1, 256>>>(out, cyc, 0.999, 0.001, n);
  k<<<1, 256>>>(out, cyc, 0.999, 0.001, n);
  cudaDeviceSynchronize();
  const char* names[] = {"DFMA", "DADD", "shfl.f64+DADD", "LDS (chase)", "bar.sync 224", "sqrt f64",
                         "div f64", "drcp_rn", "__syncthreads 256", "smem flag round trip"};
  for (int i = 0; i < 10; ++i) printf("%-22s %7.1f cycles\n", names[i], (double)cyc[i] / n);
  int clk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("clock %d kHz\n", clk);
  return 0;
}
