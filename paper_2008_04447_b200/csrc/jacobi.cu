// One-sided (Hestenes) Jacobi SVD of a small dense matrix on the device: the
// reference's deterministic k x k SVD used by tuxv(refine_sigma=True)
// (randomized.py:401-403 -> jacobi.py:50-117) and by the quality harness.
//
// Same method as the reference: round-robin tournament rounds of disjoint
// column pairs (jacobi.py:24-37; player at seat i of round r is 0 for i = 0,
// else 1 + ((i - 1 - r) mod (q - 1)), which is the reference's rotation of
// seats 1..q-1), a pair rotates when |gamma| > 1e-15 sqrt(alpha beta)
// (jacobi.py:75), the rotation angle of jacobi.py:84-88, up to 60 sweeps,
// stop after a sweep with no rotation.  One CTA: a warp per pair (pairs of a
// round are disjoint, so the round is one batched rotation as in the
// reference), a block barrier between rounds.  Column norms and the stable
// descending order of the singular values close the kernel.
#include <algorithm>

#include "common.cuh"

namespace sqr {
namespace {

constexpr int kJThreads = 1024;
constexpr int kJWarps = kJThreads / 32;
constexpr double kPairTol = 1e-15;

__device__ __forceinline__ int seat_player(int i, int r, int q) {
  return i == 0 ? 0 : 1 + ((i - 1 - r) % (q - 1) + (q - 1)) % (q - 1);
}

__global__ void __launch_bounds__(kJThreads) jacobi_kernel(double* __restrict__ W, int64_t ldw, int m, int n,
                                                           double* __restrict__ V, int64_t ldv,
                                                           double* __restrict__ sigma, int64_t* __restrict__ order,
                                                           int max_sweeps, int32_t* __restrict__ info) {
  __shared__ int rotated;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // V = I
  for (int64_t e = threadIdx.x; e < (int64_t)n * n; e += blockDim.x) {
    const int r = (int)(e % n), c = (int)(e / n);
    V[c * ldv + r] = r == c ? 1.0 : 0.0;
  }
  const int q = n + (n & 1);  // seats (a dummy player n when n is odd)
  int sweeps = 0;
  bool converged = false;
  __syncthreads();
  for (; sweeps < max_sweeps; ++sweeps) {
    if (threadIdx.x == 0) rotated = 0;
    __syncthreads();
    for (int r = 0; r < q - 1; ++r) {
      for (int pr = warp; pr < q / 2; pr += kJWarps) {
        const int i = seat_player(pr, r, q), j = seat_player(q - 1 - pr, r, q);
        if (i >= n || j >= n) continue;  // the dummy's pair
        double* wi = W + (int64_t)i * ldw;
        double* wj = W + (int64_t)j * ldw;
        double a = 0.0, b = 0.0, g = 0.0;
        for (int t = lane; t < m; t += 32) {
          const double x = wi[t], y = wj[t];
          a = fma(x, x, a);
          b = fma(y, y, b);
          g = fma(x, y, g);
        }
        a = warp_sum(a);
        b = warp_sum(b);
        g = warp_sum(g);
        if (!(fabs(g) > kPairTol * sqrt(a * b))) continue;
        const double zeta = (b - a) / (2.0 * g);
        double t = zeta == 0.0 ? 1.0 : copysign(1.0, zeta) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
        const double c = 1.0 / sqrt(1.0 + t * t), s = c * t;
        for (int e = lane; e < m; e += 32) {
          const double x = wi[e], y = wj[e];
          wi[e] = c * x - s * y;
          wj[e] = s * x + c * y;
        }
        double* vi = V + (int64_t)i * ldv;
        double* vj = V + (int64_t)j * ldv;
        for (int e = lane; e < n; e += 32) {
          const double x = vi[e], y = vj[e];
          vi[e] = c * x - s * y;
          vj[e] = s * x + c * y;
        }
        if (lane == 0) rotated = 1;
      }
      __syncthreads();
    }
    if (!rotated) {
      converged = true;
      break;
    }
    __syncthreads();
  }
  // singular values = column norms; stable descending order (jacobi.py:107-110)
  for (int c = warp; c < n; c += kJWarps) {
    const double* w = W + (int64_t)c * ldw;
    double a = 0.0;
    for (int t = lane; t < m; t += 32) a = fma(w[t], w[t], a);
    a = warp_sum(a);
    if (lane == 0) sigma[c] = sqrt(a);
  }
  __syncthreads();
  for (int c = threadIdx.x; c < n; c += blockDim.x) {
    const double v = sigma[c];
    int rank = 0;
    for (int o = 0; o < n; ++o) {
      const double u = sigma[o];
      rank += (u > v || (u == v && o < c)) ? 1 : 0;
    }
    order[rank] = c;
  }
  if (threadIdx.x == 0) {
    info[0] = converged ? sweeps + 1 : -1;
    info[1] = n;
  }
}

}  // namespace
}  // namespace sqr

using namespace sqr;

// W (m x n, m >= n, ld ldw) is rotated in place into W V; V (n x n, ldv)
// receives the accumulated rotations; sigma[c] = ||W[:, c]|| (unsorted) and
// order[] the stable descending order of sigma; info[0] = sweeps used (the
// converging sweep included), -1 when max_sweeps did not converge
// (jacobi.py:104-105 raises LinAlgError).
extern "C" int sqr_jacobi_svd(double* W, int64_t ldw, int64_t m, int64_t n, double* V, int64_t ldv, double* sigma,
                              int64_t* order, int max_sweeps, int32_t* info, void* stream) {
  if (n <= 0) return SQR_OK;
  if (W == nullptr || V == nullptr || sigma == nullptr || order == nullptr || info == nullptr || m < n ||
      ldw < m || ldv < n || n > 4096 || max_sweeps < 1) {
    set_error("sqr_jacobi_svd: need m >= n, n <= 4096 (jacobi.py:54-55) and valid buffers");
    return SQR_EINVAL;
  }
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  ProfScope ps(kTagMisc, s);
  jacobi_kernel<<<1, kJThreads, 0, s>>>(W, ldw, (int)m, (int)n, V, ldv, sigma, order, max_sweeps, info);
  SQR_LAUNCH("jacobi_kernel");
  return SQR_OK;
}
