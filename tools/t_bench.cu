// Latency of the 32x32 compact-WY T recurrence on one warp (builder tool).
//   T[i][c] = -tau_c sum_{l<c} T[i][l] G[l][c],  T[i][i] = tau_i
// V1: lane i keeps row i, G column c loaded per step as LDS.128 broadcasts.
// V2: same, all 32 columns' partial sums accumulated right-looking:
//     after T[i][c] is known, p[c'] += T[i][c] G[c][c'] for c' > c
//     (G row c, contiguous) -> one FMA per future column, no reduction chain.
#include <cstdio>
#include <cuda_runtime.h>

template <int V>
__global__ void tb(const double* Gg, const double* tg, double* out, long long* cyc) {
  __shared__ __align__(16) double Gs[32 * 32];
  __shared__ double taus[32];
  const int lane = threadIdx.x;
  for (int e = lane; e < 1024; e += 32) Gs[e] = Gg[e];
  taus[lane] = tg[lane];
  __syncwarp();
  long long t0 = clock64();
  double tr[32];
  if (V == 1) {
#pragma unroll
    for (int c = 0; c < 32; ++c) {
      const double2* Gc = reinterpret_cast<const double2*>(Gs + c * 32);  // G[:, c] contiguous
      double2 gv[16];
#pragma unroll
      for (int l2 = 0; l2 < (c + 1) / 2; ++l2) gv[l2] = Gc[l2];
      double s0 = 0, s1 = 0, s2 = 0, s3 = 0;
#pragma unroll
      for (int l2 = 0; l2 < (c + 1) / 2; ++l2) {
        const int l = 2 * l2;
        if (l2 & 1) {
          s2 = fma(tr[l], gv[l2].x, s2);
          if (l + 1 < c) s3 = fma(tr[l + 1], gv[l2].y, s3);
        } else {
          s0 = fma(tr[l], gv[l2].x, s0);
          if (l + 1 < c) s1 = fma(tr[l + 1], gv[l2].y, s1);
        }
      }
      const double tc = taus[c];
      tr[c] = c == lane ? tc : (c > lane ? -tc * ((s0 + s1) + (s2 + s3)) : 0.0);
    }
  } else {
    double p[32];
#pragma unroll
    for (int c = 0; c < 32; ++c) p[c] = 0.0;
#pragma unroll
    for (int c = 0; c < 32; ++c) {
      const double tc = taus[c];
      tr[c] = c == lane ? tc : (c > lane ? -tc * p[c] : 0.0);
      // fold T[i][c] into the sums of the later columns: p[c'] += T[i][c] G[c][c']
      const double2* Gr = reinterpret_cast<const double2*>(Gs + c * 32);  // symmetric: row c == column c
#pragma unroll
      for (int c2 = (c + 1) / 2; c2 < 16; ++c2) {
        const double2 gv = Gr[c2];
        if (2 * c2 > c) p[2 * c2] = fma(tr[c], gv.x, p[2 * c2]);
        p[2 * c2 + 1] = fma(tr[c], gv.y, p[2 * c2 + 1]);
      }
    }
  }
  long long t1 = clock64();
  for (int c = 0; c < 32; ++c) out[lane * 32 + c] = tr[c];
  if (lane == 0) cyc[V] = t1 - t0;
}

int main() {
  double *G, *t, *o;
  long long* cyc;
  cudaMalloc(&G, 8192);
  cudaMalloc(&t, 256);
  cudaMalloc(&o, 8192 * 2);
  cudaMalloc(&cyc, 64);
  double hG[1024], ht[32];
  for (int i = 0; i < 32; ++i) {
    ht[i] = 1.0 + 0.01 * i;
    for (int j = 0; j < 32; ++j) hG[i * 32 + j] = (i == j) ? 1.0 : 0.01 * ((i * 7 + j * 3) % 11 - 5);
  }
  for (int i = 0; i < 32; ++i)
    for (int j = 0; j < i; ++j) hG[i * 32 + j] = hG[j * 32 + i];
  cudaMemcpy(G, hG, 8192, cudaMemcpyHostToDevice);
  cudaMemcpy(t, ht, 256, cudaMemcpyHostToDevice);
  for (int r = 0; r < 3; ++r) {
    tb<1><<<1, 32>>>(G, t, o, cyc);
    tb<2><<<1, 32>>>(G, t, o + 1024, cyc);
  }
  long long hc[4];
  cudaMemcpy(hc, cyc, 32, cudaMemcpyDeviceToHost);
  double ho[2048];
  cudaMemcpy(ho, o, 16384, cudaMemcpyDeviceToHost);
  double md = 0;
  for (int i = 0; i < 1024; ++i) md = fmax(md, fabs(ho[i] - ho[1024 + i]));
  printf("V1 %lld cycles, V2 %lld cycles, max diff %.3e\n", hc[1], hc[2], md);
  return 0;
}
